timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
bash tools/xcheck.sh
for a in "--cfg 1" "--cfg 3 --B 256 --reps 3" "--cfg 4" "--cfg 2" "--cfg 4 --c64" "--cfg 2 --c64"; do python tools/prof_accel.py $a --reps 5; done
python tools/stream_flush_ab.py 1; python tools/stream_flush_ab.py 3
