#!/bin/bash
# build, bitmap-path parity tests, one bench line summarised (GPU box helper)
make -C paper_2406_03726_b200/csrc -s >/dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -k "${TESTS:-bitmap or fuzz or golden}" -x -q 2>&1 | tail -2
for c in ${CONFIGS:-1}; do
python bench.py --config $c --steps ${STEPS:-50} --warmup 5 --no-cpu-baseline --no-e2e --force-path ${FORCE:-0} > gpurun_out/b$c.log 2>&1
tail -1 gpurun_out/b$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg', $c, round(d['ms_per_step']*1e3,1), 'us', [(r['kernel'], round(r['ms_per_launch']*1e3,1)) for r in d.get('kernels', [])][:8])"
done
