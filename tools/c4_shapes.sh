# K2 cluster shapes for config 4 (M8, J=4096) and config 2 (M2, J=20000):
# CTAs per bin (CL), slots per thread, constants in registers (SMEM 0) or smem (1)
for r in 1 2; do
python tools/prof_accel.py --cfg 4 --reps 3
RCSCM_ACCEL_CL=2 RCSCM_ACCEL_SMEM=1 python tools/prof_accel.py --cfg 4 --reps 3
RCSCM_ACCEL_CL=4 RCSCM_ACCEL_SMEM=1 python tools/prof_accel.py --cfg 4 --reps 3
RCSCM_ACCEL_CL=8 RCSCM_ACCEL_SMEM=1 python tools/prof_accel.py --cfg 4 --reps 3
done
python tools/prof_accel.py --cfg 2 --reps 3
RCSCM_ACCEL_CL=16 RCSCM_ACCEL_SMEM=0 python tools/prof_accel.py --cfg 2 --reps 3
