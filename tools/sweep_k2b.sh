for I in 148 296 444; do python tools/prof_accel.py --I $I --reps 5; done
for I in 148 444; do RCSCM_ACCEL_MINB=1 python tools/prof_accel.py --I $I --reps 5; done
python tools/prof_accel.py --I 148 --J 320 --reps 5
python tools/prof_accel.py --I 444 --J 320 --reps 5
python tools/prof_accel.py --I 888 --J 320 --reps 5
RCSCM_ACCEL_SPT=4 python tools/prof_accel.py --I 444 --reps 5
RCSCM_ACCEL_SPT=6 python tools/prof_accel.py --I 444 --reps 5
RCSCM_ACCEL_SPT=8 python tools/prof_accel.py --I 444 --reps 5
RCSCM_ACCEL_SPT=8 python tools/prof_accel.py --I 1025 --reps 5
