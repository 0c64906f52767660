# A/B of library builds on the C3 batch: bash tools/gpu_ab_c3.sh name1 name2 ... (main = the in-tree build)
for rep in 1 2; do
  for n in "$@"; do
    if [ "$n" = main ]; then lib=""; else lib=$PWD/build/ab/$n/librcscm_gpu.so; fi
    echo -n "$n: "; RCSCM_GPU_LIB=$lib timeout 300 python tools/prof_accel.py --cfg 3 --B 128 --reps 5 2>&1 | tail -1
  done
done
