# A/B of stream embed debug variants (bench.py --stream-variant V) on configs
for c in ${CONFIGS:-3 4 2}; do for v in ${VARIANTS:-0 1}; do
timeout 300 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --stream-variant $v > gpurun_out/av_${c}_${v}.json 2>/dev/null
done; done
