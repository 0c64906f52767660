# config 2 (J=20000): 512-thread CTAs, one per SM, in 8-CTA clusters (RCSCM_ACCEL_NT512)
python tools/prof_accel.py --cfg 2 --reps 3
RCSCM_ACCEL_NT512=1 RCSCM_ACCEL_SPT=5 python tools/prof_accel.py --cfg 2 --reps 3
RCSCM_ACCEL_NT512=1 RCSCM_ACCEL_SPT=6 python tools/prof_accel.py --cfg 2 --reps 3
RCSCM_ACCEL_NT512=1 RCSCM_ACCEL_CL=16 RCSCM_ACCEL_SPT=3 python tools/prof_accel.py --cfg 2 --reps 3
