for v in "X=1" "RCSCM_ACCEL_SMEM=2 RCSCM_ACCEL_MINB=4" "RCSCM_ACCEL_SMEM=1 RCSCM_ACCEL_MINB=4" "RCSCM_ACCEL_SMEM=2 RCSCM_ACCEL_MINB=5" "RCSCM_ACCEL_DIRECT=0"; do
  echo "$v"; env $v python tools/prof_accel.py --reps 5
done
