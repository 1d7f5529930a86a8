# Round-end ncu evidence for configs[3] (run under gpurun, one GPU):
#   1. the launch list of a short bench run (cold-cache per-launch times),
#   2. one `--set full` capture of every k_st_* kernel of one encode.
set -x
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p_plain.json 2> gpurun_out/p_plain.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p_launches.csv \
  python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p_launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'k_st_|k_label' -c 12 \
  -o gpurun_out/p_full_c3 -f python tools/encode_once.py 3 1 > gpurun_out/p_full.log 2>&1
