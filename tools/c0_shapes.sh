# config 0 (M2, I513, J320) K2 shapes: slots per thread (threads per bin = 320 / SPT)
python tools/prof_accel.py --cfg 0 --reps 5
for spt in 2 3 4 8; do RCSCM_ACCEL_SPT=$spt python tools/prof_accel.py --cfg 0 --reps 5; done
RCSCM_FUSE_PRE=0 python tools/prof_accel.py --cfg 0 --reps 5
