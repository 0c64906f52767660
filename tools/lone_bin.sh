for spt in 5 4 3; do RCSCM_ACCEL_SPT=$spt python tools/prof_accel.py --I 148 --unfused --reps 5; done
for cl in 2 4; do RCSCM_ACCEL_CL=$cl python tools/prof_accel.py --I 148 --unfused --reps 5; done
for I in 148 296 444 888 1025; do python tools/prof_accel.py --I $I --unfused --reps 5; done
