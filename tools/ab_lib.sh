# A/B of two builds of libgee.so on one GPU: the in-tree library, then abtest/libgee_A.so copied over it.
# CFGS="3 4 2" bash tools/ab_lib.sh
timeout 900 python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -1
for lib in B A; do
  if [ $lib = A ]; then cp abtest/libgee_A.so paper_2406_03726_b200/libgee.so; fi
  for c in ${CFGS:-3 4 2}; do
    PYTHONFAULTHANDLER=1 timeout -s SEGV 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/al_${lib}_c${c}.json 2> gpurun_out/al_${lib}_c${c}.err
    python tools/ab_show.py gpurun_out/al_${lib}_c${c}.json 2>/dev/null || tail -3 gpurun_out/al_${lib}_c${c}.err
  done
done
