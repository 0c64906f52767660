./build/k2_cluster_probe 2>&1 | grep -v "^  sm" | tee gpurun_out/k2_cluster_probe_stas.txt
for a in "--cfg 1" "--cfg 4" "--cfg 2" "--cfg 4 --c64" "--cfg 2 --c64"; do python tools/prof_accel.py $a --reps 5; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
