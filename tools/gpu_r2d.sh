# NaN bit patterns, cluster-K2 phase probe, NaN tests, K2 timings
./build/nan_probe | tee gpurun_out/nan_probe.txt
./build/k2_cluster_probe | tee gpurun_out/k2_cluster_probe.txt
timeout 900 python -m pytest tests/test_gpu_full.py -q -k nan 2>&1 | tail -3
for a in "--cfg 1" "--cfg 3 --B 32" "--cfg 4" "--cfg 2"; do python tools/prof_accel.py $a --reps 5; done
