# config 1 K2 (unfused, so every variant is comparable) at 3 / 4 / 5 CTAs per SM:
# registers (SMEM 0, MINB 3) vs constants in shared memory (SMEM 1 / 2, MINB 4 / 5)
export RCSCM_FUSE_PRE=0
for r in 1 2; do
python tools/prof_accel.py --cfg 1 --reps 10 --unfused
RCSCM_ACCEL_SMEM=1 RCSCM_ACCEL_MINB=4 python tools/prof_accel.py --cfg 1 --reps 10 --unfused
RCSCM_ACCEL_SMEM=2 RCSCM_ACCEL_MINB=4 python tools/prof_accel.py --cfg 1 --reps 10 --unfused
RCSCM_ACCEL_SMEM=2 RCSCM_ACCEL_MINB=5 python tools/prof_accel.py --cfg 1 --reps 10 --unfused
done
