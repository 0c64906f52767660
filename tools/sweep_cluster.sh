# cluster-path (large J) K2 configuration sweep: cfg4 (J=4096, M=8) and cfg2 (J=20000)
for cl in 2 4 8 16; do for sm in 0 1; do for spt in 2 4 5 8; do
  echo "cfg4 CL=$cl SMEM=$sm SPT=$spt"; RCSCM_ACCEL_CL=$cl RCSCM_ACCEL_SMEM=$sm RCSCM_ACCEL_SPT=$spt timeout 60 python tools/prof_accel.py --cfg 4 --I 512 --reps 3 2>&1 | tail -1
done; done; done
for cl in 16; do for sm in 0 1; do for spt in 4 5 6 8; do
  echo "cfg2 CL=$cl SMEM=$sm SPT=$spt"; RCSCM_ACCEL_CL=$cl RCSCM_ACCEL_SMEM=$sm RCSCM_ACCEL_SPT=$spt timeout 60 python tools/prof_accel.py --cfg 2 --I 256 --reps 3 2>&1 | tail -1
done; done; done
