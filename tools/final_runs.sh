# Round-end measurement set (GPU box): full GPU suite, bench lines, reference arm,
# then the ncu evidence for configs[3] / configs[4] (launch list + --set full captures).
set -x
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/final_gputests.txt
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/final_cfg3.json 2> gpurun_out/final_cfg3.err
timeout 300 python bench.py --steps 20 --warmup 3 --fp32 --no-cpu-baseline > gpurun_out/final_cfg3_fp32.json 2> gpurun_out/final_cfg3_fp32.err
for c in 0 1 2 4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/final_cfg$c.json 2> gpurun_out/final_cfg$c.err
done
timeout 1200 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/final_ref_cfg3.json 2> gpurun_out/final_ref_cfg3.err
bash tools/prof_embed.sh final
