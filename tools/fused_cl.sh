# cluster shapes with the sigma / tau precompute fused into K2 (default) vs K1 + K2
for r in 1 2; do
python tools/prof_accel.py --cfg 4 --reps 3
RCSCM_FUSE_PRE=0 python tools/prof_accel.py --cfg 4 --reps 3
python tools/prof_accel.py --cfg 2 --reps 3
RCSCM_FUSE_PRE=0 python tools/prof_accel.py --cfg 2 --reps 3
done
