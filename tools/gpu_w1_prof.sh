# the one-warp K2 on C3: GPU tests, bench, ncu capture (after the bench ran clean)
mkdir -p gpurun_out/r02d
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02d/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02d/pytest.log
timeout 900 python bench.py > gpurun_out/r02d/bench.json 2> gpurun_out/r02d/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -c 1 --launch-skip 5 -k regex:k_accel -o gpurun_out/r02d/k_accel_c3 python tools/prof_accel.py --cfg 3 --B 256 --reps 1 > gpurun_out/r02d/ncu.log 2>&1
cp profiles/ncu_summary.json gpurun_out/r02d/
NCU_SUMMARY_DIR=gpurun_out/r02d python tools/ncu_summary.py k_accel_c3=gpurun_out/r02d/k_accel_c3.ncu-rep@k_accel > /dev/null
ncu -i gpurun_out/r02d/k_accel_c3.ncu-rep --page source --csv --print-source sass > gpurun_out/r02d/k_accel_c3_sass.csv 2>/dev/null
ncu -i gpurun_out/r02d/k_accel_c3.ncu-rep --page details --csv > gpurun_out/r02d/k_accel_c3_details.csv 2>/dev/null
tail -3 gpurun_out/r02d/pytest.log
