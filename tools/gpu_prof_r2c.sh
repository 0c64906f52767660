# round-2 ncu captures of K2 after the scalar-state change (each command ran clean
# without ncu first, in the bench and A/B runs): C3 headline (256 utterances), C1,
# C4, C2; the headline's source page; then the bench's launch list.
set -x
mkdir -p /tmp/ncu gpurun_out/r02c
N="ncu --set full --clock-control none --import-source on -c 1 --launch-skip 5"
timeout 900 $N -k regex:k_accel -o /tmp/ncu/k_accel_c3 python tools/prof_accel.py --cfg 3 --B 256 --reps 1 > gpurun_out/r02c/ncu_full.log 2>&1
timeout 900 $N -k regex:k_accel -o /tmp/ncu/k_accel_c1 python tools/prof_accel.py --cfg 1 --reps 1 >> gpurun_out/r02c/ncu_full.log 2>&1
timeout 900 $N -k regex:k_accel -o /tmp/ncu/k_accel_c4 python tools/prof_accel.py --cfg 4 --reps 1 >> gpurun_out/r02c/ncu_full.log 2>&1
timeout 900 $N -k regex:k_accel -o /tmp/ncu/k_accel_c2 python tools/prof_accel.py --cfg 2 --reps 1 >> gpurun_out/r02c/ncu_full.log 2>&1
cp profiles/ncu_summary.json gpurun_out/r02c/
NCU_SUMMARY_DIR=gpurun_out/r02c python tools/ncu_summary.py k_accel_c3=/tmp/ncu/k_accel_c3.ncu-rep@k_accel \
  k_accel_c1=/tmp/ncu/k_accel_c1.ncu-rep@k_accel k_accel_c4=/tmp/ncu/k_accel_c4.ncu-rep@k_accel \
  k_accel_c2=/tmp/ncu/k_accel_c2.ncu-rep@k_accel > /dev/null
ncu -i /tmp/ncu/k_accel_c3.ncu-rep --page source --csv --print-source sass > gpurun_out/r02c/k_accel_c3_sass.csv 2>/dev/null
ncu -i /tmp/ncu/k_accel_c3.ncu-rep --page details --csv > gpurun_out/r02c/k_accel_c3_details.csv 2>/dev/null
cp /tmp/ncu/k_accel_c3.ncu-rep /tmp/ncu/k_accel_c4.ncu-rep gpurun_out/r02c/ 2>/dev/null
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02c/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r02c/ncu_launch.log 2>&1
du -sh gpurun_out
