# A/B of library builds on the cluster K2 shapes: bash tools/gpu_ab2.sh name1 name2 ...
for rep in 1 2; do
for n in "$@"; do
  if [ "$n" = main ]; then lib=""; else lib=$PWD/build/ab/$n/librcscm_gpu.so; fi
  for a in "--cfg 4" "--cfg 2"; do
    echo -n "$n: "; RCSCM_GPU_LIB=$lib python tools/prof_accel.py $a --reps 5
  done
done
done
