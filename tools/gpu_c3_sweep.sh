# C3 (128 utterances) shape / unroll sweep: bash tools/gpu_c3_sweep.sh
for n in main un1 un3; do
  if [ "$n" = main ]; then lib=""; else lib=$PWD/build/ab/$n/librcscm_gpu.so; fi
  echo -n "$n: "; RCSCM_GPU_LIB=$lib timeout 300 python tools/prof_accel.py --cfg 3 --B 128 --reps 5 2>&1 | tail -1
done
for spt in 4 3 2 6; do
  echo -n "spt=$spt: "; RCSCM_ACCEL_SPT=$spt timeout 300 python tools/prof_accel.py --cfg 3 --B 128 --reps 5 2>&1 | tail -1
done
