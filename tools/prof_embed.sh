# ncu evidence for the stream encode (one GPU, run under gpurun):
#   launch list of a short configs[3] bench run, then one --set full capture
#   of the k_st_* passes at configs[3] and of k_st_embed at configs[4].
set -x
tag=${1:-p}
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_plain.json 2> gpurun_out/${tag}_plain.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_st_embed|k_st_degree|k_st_part1|k_st_part2|k_st_hist' -c 6 \
  -o gpurun_out/${tag}_full_c3 -f python tools/encode_once.py 3 1 > gpurun_out/${tag}_full_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_st_embed' -c 1 \
  -o gpurun_out/${tag}_full_c4 -f python tools/encode_once.py 4 1 > gpurun_out/${tag}_full_c4.log 2>&1
ls -la gpurun_out
