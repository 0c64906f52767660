# K2d (two bins in flight per cluster): its tests, then an A/B against k_accel on C4
# and on a ragged M = 2 shape, then the whole GPU suite with K2d enabled
mkdir -p gpurun_out/r2m
timeout 900 python -m pytest tests/test_gpu_db.py -x -q > gpurun_out/r2m/pytest_db.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2m/pytest_db.log
tail -5 gpurun_out/r2m/pytest_db.log
for rep in 1 2; do
  for db in 0 1; do
    for a in "--cfg 4" "--cfg 4 --I 512" "--cfg 0 --J 3000" "--cfg 1 --J 8000"; do
      echo -n "db=$db: "; RCSCM_ACCEL_DB=$db timeout 300 python tools/prof_accel.py $a --reps 5 2>&1 | tail -1
    done
  done
done | tee gpurun_out/r2m/ab.txt
RCSCM_ACCEL_DB=1 timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2m/pytest_gpu_db1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2m/pytest_gpu_db1.log
tail -3 gpurun_out/r2m/pytest_gpu_db1.log
