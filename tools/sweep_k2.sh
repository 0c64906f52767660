# K2 sweep: wave fill (I) x launch variants. Usage: bash tools/sweep_k2.sh > gpurun_out/sweep.log
for I in 444 888 1025 1036 1184 1332; do
  python tools/prof_accel.py --I $I --reps 5
done
for v in "RCSCM_ACCEL_SMEM=2 RCSCM_ACCEL_MINB=4" "RCSCM_ACCEL_SMEM=1 RCSCM_ACCEL_MINB=4" "RCSCM_ACCEL_SMEM=2 RCSCM_ACCEL_MINB=5"; do
  for I in 592 1025 1184; do
    echo "$v"; env $v python tools/prof_accel.py --I $I --reps 5
  done
done
