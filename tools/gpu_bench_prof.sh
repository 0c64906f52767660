# bench line + launch list + ncu --set full of K2/K1/K4/K3 (run under gpurun; outputs in gpurun_out/)
set -x
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_accel -c 1 -o gpurun_out/k_accel python tools/prof_accel.py --reps 2 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_accel -c 1 -o gpurun_out/k_accel_c64 python tools/prof_accel.py --reps 2 --c64 >> gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_slots -c 1 -o gpurun_out/k_slots python tools/prof_accel.py --reps 1 >> gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wiener -c 1 -o gpurun_out/k_wiener python tools/prof_accel.py --reps 1 --wiener >> gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_naive -c 1 -o gpurun_out/k_naive python tools/prof_accel.py --reps 1 --naive >> gpurun_out/ncu_full.log 2>&1
cat gpurun_out/bench.json
