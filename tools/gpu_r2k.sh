# 512-thread CTAs (k_accel MINB = -1): C4 as one CTA per bin, C2 as 5-CTA clusters
mkdir -p gpurun_out/r2k
for rep in 1 2; do
  for big in 0 1; do
    for a in "--cfg 4" "--cfg 2"; do
      echo -n "big=$big: "; RCSCM_ACCEL_BIG=$big timeout 300 python tools/prof_accel.py $a --reps 5 2>&1 | tail -1
    done
  done
done | tee gpurun_out/r2k/ab.txt
RCSCM_ACCEL_BIG=1 timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2k/pytest_gpu_big.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2k/pytest_gpu_big.log
tail -3 gpurun_out/r2k/pytest_gpu_big.log
