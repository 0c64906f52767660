# A/B of library builds on the single-CTA shapes (C0, C1, C3 fused and unfused): bash tools/gpu_ab_single.sh name1 ...
for rep in 1 2; do
  for n in "$@"; do
    if [ "$n" = main ]; then lib=""; else lib=$PWD/build/ab/$n/librcscm_gpu.so; fi
    for a in "--cfg 3 --B 128" "--cfg 3 --B 128 --unfused" "--cfg 1" "--cfg 0"; do
      echo -n "$n $a: "; RCSCM_GPU_LIB=$lib timeout 300 python tools/prof_accel.py $a --reps 5 2>&1 | tail -1
    done
  done
done
