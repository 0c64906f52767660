# round-2 ncu captures (each after its command ran clean without ncu):
#   full-set captures of K2 on C3 (headline), C1, C4, C2, the C3 stream kernels and
#   k_naive, then the bench's launch list. Reports stay in /tmp/ncu on the box;
#   summaries (raw-page metrics, source-page CSV of the headline K2) come back.
set -x
mkdir -p /tmp/ncu gpurun_out/r02
N="ncu --set full --clock-control none --import-source on -c 1 --launch-skip 5"
python tools/prof_accel.py --cfg 3 --B 256 --reps 1 > gpurun_out/r02/plain.log 2>&1
timeout 900 $N -k regex:k_accel -o /tmp/ncu/k_accel_c3 python tools/prof_accel.py --cfg 3 --B 256 --reps 1 > gpurun_out/r02/ncu_full.log 2>&1
timeout 900 $N -k regex:k_accel -o /tmp/ncu/k_accel_c1 python tools/prof_accel.py --cfg 1 --reps 1 >> gpurun_out/r02/ncu_full.log 2>&1
timeout 900 $N -k regex:k_accel -o /tmp/ncu/k_accel_c4 python tools/prof_accel.py --cfg 4 --reps 1 >> gpurun_out/r02/ncu_full.log 2>&1
timeout 900 $N -k regex:k_accel -o /tmp/ncu/k_accel_c2 python tools/prof_accel.py --cfg 2 --reps 1 >> gpurun_out/r02/ncu_full.log 2>&1
timeout 900 $N -k regex:k_pre -o /tmp/ncu/k_pre_c3 python tools/prof_accel.py --cfg 3 --B 256 --reps 1 --unfused >> gpurun_out/r02/ncu_full.log 2>&1
timeout 900 $N -k regex:k_wiener -o /tmp/ncu/k_wiener_c3 python tools/prof_accel.py --cfg 3 --B 256 --reps 1 --wiener >> gpurun_out/r02/ncu_full.log 2>&1
timeout 900 $N -k regex:k_naive -o /tmp/ncu/k_naive_c3 python tools/prof_accel.py --cfg 3 --B 32 --reps 1 --naive >> gpurun_out/r02/ncu_full.log 2>&1
NCU_SUMMARY_DIR=gpurun_out/r02 python tools/ncu_summary.py k_accel_c3=/tmp/ncu/k_accel_c3.ncu-rep@k_accel \
  k_accel_c1=/tmp/ncu/k_accel_c1.ncu-rep@k_accel k_accel_c4=/tmp/ncu/k_accel_c4.ncu-rep@k_accel \
  k_accel_c2=/tmp/ncu/k_accel_c2.ncu-rep@k_accel k_pre_c3=/tmp/ncu/k_pre_c3.ncu-rep@k_pre \
  k_wiener_c3=/tmp/ncu/k_wiener_c3.ncu-rep@k_wiener k_naive_c3=/tmp/ncu/k_naive_c3.ncu-rep@k_naive > /dev/null
ncu -i /tmp/ncu/k_accel_c3.ncu-rep --page source --csv > gpurun_out/r02/k_accel_c3_source.csv 2>/dev/null
ncu -i /tmp/ncu/k_accel_c3.ncu-rep --page details --csv > gpurun_out/r02/k_accel_c3_details.csv 2>/dev/null
ls -la /tmp/ncu
cp /tmp/ncu/k_accel_c3.ncu-rep gpurun_out/r02/ 2>/dev/null
du -sh gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r02/ncu_launch.log 2>&1
du -sh gpurun_out
