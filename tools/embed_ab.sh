#!/bin/bash
# A/B of the K > 8 embed variants (GPU box helper):
#   CONFIGS="2 3 4" BUDGETS="0 4096 12288" ROWMAX="256" bash tools/embed_ab.sh
for c in ${CONFIGS:-2 3 4}; do
for b in ${BUDGETS:-0 12288}; do
for m in ${ROWMAX:-256}; do
python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e --embed-flat-bytes $b --embed-flat-rowmax $m > gpurun_out/ab_c${c}_b${b}_m$m.log 2>&1
tail -1 gpurun_out/ab_c${c}_b${b}_m$m.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=dict((r['kernel'], r['ms_per_launch']) for r in d.get('kernels', [])); print('cfg', $c, 'flat', $b, 'rowmax', $m, round(d['ms_per_step'],3), 'ms  k_embed', round(k.get('k_embed', -1), 3))" || tail -3 gpurun_out/ab_c${c}_b${b}_m$m.log
done; done; done
