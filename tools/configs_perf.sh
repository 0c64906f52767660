# K2 step (fused when possible) on every BASELINE config shape, c128 and c64 for config 4
python tools/prof_accel.py --cfg 0 --reps 3
python tools/prof_accel.py --cfg 1 --reps 3
python tools/prof_accel.py --cfg 2 --reps 3
python tools/prof_accel.py --cfg 3 --B 32 --reps 3
python tools/prof_accel.py --cfg 4 --reps 3
python tools/prof_accel.py --cfg 4 --reps 3 --c64
