# SST2 (folded scalar-state arithmetic): the GPU suite on the new build, then an
# A/B against the previous arithmetic (build/ab/sst1) on every config
mkdir -p gpurun_out/r2i
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2i/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2i/pytest_gpu.log
tail -3 gpurun_out/r2i/pytest_gpu.log
for rep in 1 2; do
  for n in main sst1; do
    if [ "$n" = main ]; then lib=""; else lib=$PWD/build/ab/$n/librcscm_gpu.so; fi
    for a in "--cfg 3 --B 128" "--cfg 4" "--cfg 2" "--cfg 1" "--cfg 0"; do
      echo -n "$n: "; RCSCM_GPU_LIB=$lib timeout 300 python tools/prof_accel.py $a --reps 5 2>&1 | tail -1
    done
  done
done | tee gpurun_out/r2i/ab.txt
