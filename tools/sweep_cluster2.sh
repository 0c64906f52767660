for d in 1 0; do
  echo "DIRECT=$d"; RCSCM_ACCEL_DIRECT=$d python tools/prof_accel.py --cfg 4 --reps 3 | tail -1
  RCSCM_ACCEL_DIRECT=$d python tools/prof_accel.py --cfg 2 --reps 3 | tail -1
  for sm in 0 1; do for spt in 5 8; do echo "cfg2 SMEM=$sm SPT=$spt"; RCSCM_ACCEL_DIRECT=$d RCSCM_ACCEL_SMEM=$sm RCSCM_ACCEL_SPT=$spt python tools/prof_accel.py --cfg 2 --I 256 --reps 3 | tail -1; done; done
  for sm in 0 1; do echo "cfg4 CL2 SMEM=$sm"; RCSCM_ACCEL_DIRECT=$d RCSCM_ACCEL_SMEM=$sm python tools/prof_accel.py --cfg 4 --I 512 --reps 3 | tail -1; done
done
