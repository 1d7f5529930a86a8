set -x
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/ref_cfg3.json 2> gpurun_out/ref_cfg3.err
timeout 300 python bench.py --fp32 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_fp32.json 2> gpurun_out/b_fp32.err
for v in "" "--permute-edges" "--weighted" "--permute-edges --weighted"; do
  tag=$(echo "$v" | tr -d ' -'); timeout 300 python bench.py --config 1 --steps 20 --warmup 3 --cpu-budget-s 4 $v > gpurun_out/b_c1_$tag.json 2> gpurun_out/b_c1_$tag.err
done
bash tools/harness_demo.sh
