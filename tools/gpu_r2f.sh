./build/k2_cluster_probe 2>&1 | grep -v "^  sm"
for a in "--cfg 1" "--cfg 3 --B 32" "--cfg 4" "--cfg 2" "--cfg 0"; do python tools/prof_accel.py $a --reps 5; done
for a in "--cfg 1" "--cfg 3 --B 32" "--cfg 0"; do RCSCM_ACCEL_MINB=4 python tools/prof_accel.py $a --reps 5; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python tools/truth_table.py 2>&1 | grep gpu
