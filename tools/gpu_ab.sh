# A/B of library builds on the K2 step: bash tools/gpu_ab.sh name1 name2 ... ("main" = in-tree build)
for rep in 1 2; do
for n in "$@"; do
  if [ "$n" = main ]; then lib=""; else lib=$PWD/build/ab/$n/librcscm_gpu.so; fi
  for a in "--cfg 1" "--cfg 3 --B 256 --reps 3" "--cfg 4" "--cfg 2"; do
    echo -n "$n: "; RCSCM_GPU_LIB=$lib python tools/prof_accel.py $a --reps 5
  done
done
done
