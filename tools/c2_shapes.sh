# config 2 (M2, J=20000, 50 it) K2 shapes in complex128: 16-CTA clusters x slots per thread
python tools/prof_accel.py --cfg 2 --reps 3
RCSCM_ACCEL_SPT=6 python tools/prof_accel.py --cfg 2 --reps 3
RCSCM_ACCEL_SPT=8 python tools/prof_accel.py --cfg 2 --reps 3
RCSCM_ACCEL_SPT=4 python tools/prof_accel.py --cfg 2 --reps 3
