# K2 (fused) time vs bin count at J = 640, M = 4: per-wave cost and the tail
# round of 1025 bins at 3 CTAs per SM (148 SMs)
for I in 148 296 444 592 740 888 1025 1036 1184 1332; do
  python tools/prof_accel.py --cfg 1 --I $I --reps 5
done
