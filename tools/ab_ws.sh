for c in ${CONFIGS:-3 4 2}; do for nt in ${NTS:-0 128}; do for t in ${TILES:-16 24 32}; do
timeout 300 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --stream-nt $nt --stream-tile-kb $t > gpurun_out/ws_${c}_${nt}_${t}.json 2>gpurun_out/ws_${c}_${nt}_${t}.err
done; done; done
