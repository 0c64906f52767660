# quick GPU cycle: parity suite + K2 timings
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for I in 148 444 1025; do python tools/prof_accel.py --I $I --reps 5; done
python tools/prof_accel.py --c64 --reps 5
