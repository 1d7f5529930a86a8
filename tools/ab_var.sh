# A/B of stream-variant debug knobs on configs 3, 4, 2 (one GPU): VARS="0 32" bash tools/ab_var.sh
set -x
timeout 900 python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -1
for c in ${CFGS:-3 4 2}; do
  for v in ${VARS:-0 32}; do
    PYTHONFAULTHANDLER=1 timeout -s SEGV 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --stream-variant $v > gpurun_out/av_c${c}_v${v}.json 2> gpurun_out/av_c${c}_v${v}.err
    python tools/ab_show.py gpurun_out/av_c${c}_v${v}.json 2>/dev/null || tail -3 gpurun_out/av_c${c}_v${v}.err
  done
done
