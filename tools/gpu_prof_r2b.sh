set -x
mkdir -p /tmp/ncu gpurun_out/r02b
N="ncu --set full --clock-control none --import-source on -c 1 --launch-skip 5"
timeout 900 $N -k regex:k_accel -o /tmp/ncu/k_accel_c4 python tools/prof_accel.py --cfg 4 --reps 1 > gpurun_out/r02b/ncu_full.log 2>&1
timeout 900 $N -k regex:k_accel -o /tmp/ncu/k_accel_c2 python tools/prof_accel.py --cfg 2 --reps 1 >> gpurun_out/r02b/ncu_full.log 2>&1
cp profiles/ncu_summary.json gpurun_out/r02b/
NCU_SUMMARY_DIR=gpurun_out/r02b python tools/ncu_summary.py k_accel_c4=/tmp/ncu/k_accel_c4.ncu-rep@k_accel \
  k_accel_c2=/tmp/ncu/k_accel_c2.ncu-rep@k_accel > /dev/null
