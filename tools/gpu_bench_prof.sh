# bench line + launch list + ncu --set full captures, in two parts so each
# gpurun_out/ stays under the 64 MiB copy-back limit:
#   bash tools/gpu_bench_prof.sh 1   bench, launch list, K2 (fused) and K2 (unfused)
#   bash tools/gpu_bench_prof.sh 2   K2 complex64, K1, K4, K3
set -x
N="ncu --set full --clock-control none --import-source on -c 1"
if [ "${1:-1}" = "1" ]; then
  timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
  timeout 900 $N -k regex:k_accel -o gpurun_out/k_accel python tools/prof_accel.py --reps 2 > gpurun_out/ncu_full.log 2>&1
  timeout 900 $N -k regex:k_accel -o gpurun_out/k_accel_unfused python tools/prof_accel.py --reps 2 --unfused >> gpurun_out/ncu_full.log 2>&1
else
  timeout 900 $N -k regex:k_accel -o gpurun_out/k_accel_c64 python tools/prof_accel.py --reps 2 --c64 > gpurun_out/ncu_full2.log 2>&1
  timeout 900 $N -k regex:k_pre -o gpurun_out/k_pre python tools/prof_accel.py --reps 1 --unfused >> gpurun_out/ncu_full2.log 2>&1
  timeout 900 $N -k regex:k_wiener -o gpurun_out/k_wiener python tools/prof_accel.py --reps 1 --wiener >> gpurun_out/ncu_full2.log 2>&1
  timeout 900 $N -k regex:k_naive -o gpurun_out/k_naive python tools/prof_accel.py --reps 1 --naive >> gpurun_out/ncu_full2.log 2>&1
fi
