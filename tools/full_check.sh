# Full GPU suite + the default bench line (one GPU, under gpurun).
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/fc_gputests.txt; cat gpurun_out/fc_gputests.txt
PYTHONFAULTHANDLER=1 timeout -s SEGV 900 python bench.py > gpurun_out/fc_cfg3.json 2> gpurun_out/fc_cfg3.err; echo "bench rc=$?"
python tools/ab_show.py gpurun_out/fc_cfg3.json
