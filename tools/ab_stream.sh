# A/B grid of the stream embed's CTA size and Z tile (bench.py debug knobs)
for c in ${CONFIGS:-3 4}; do for nt in ${NTS:-128 256}; do for t in ${TILES:-48 64}; do
timeout 300 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --stream-nt $nt --stream-tile-kb $t > gpurun_out/ab_${c}_${nt}_${t}.json 2>/dev/null
done; done; done
