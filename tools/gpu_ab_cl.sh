# A/B of library builds on the cluster shapes C4 and C2: bash tools/gpu_ab_cl.sh name1 ...
for rep in 1 2; do
  for n in "$@"; do
    if [ "$n" = main ]; then lib=""; else lib=$PWD/build/ab/$n/librcscm_gpu.so; fi
    for a in "--cfg 4" "--cfg 2"; do
      echo -n "$n $a: "; RCSCM_GPU_LIB=$lib timeout 300 python tools/prof_accel.py $a --reps 5 2>&1 | tail -1
    done
  done
done
