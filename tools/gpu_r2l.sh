# round-2 evidence on the SST2 build: GPU suite, truth table, bench (both arms),
# ncu --set full of K2 on C3 / C4 / C2 / C1 (each command ran clean without ncu
# first), source page of the headline, the bench's launch list, smoke
set -x
mkdir -p /tmp/ncu gpurun_out/r2l
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2l/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2l/pytest_gpu.log
timeout 900 python tools/truth_table.py > gpurun_out/r2l/parity_truth.md 2> gpurun_out/r2l/parity_truth.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2l/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2l/smoke.log
timeout 900 python bench.py > gpurun_out/r2l/bench.json 2> gpurun_out/r2l/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2l/bench_ref.json 2> gpurun_out/r2l/bench_ref.err
N="ncu --set full --clock-control none --import-source on -c 1 --launch-skip 5"
timeout 900 $N -k regex:k_accel -o /tmp/ncu/k_accel_c3 python tools/prof_accel.py --cfg 3 --B 256 --reps 1 > gpurun_out/r2l/ncu_full.log 2>&1
timeout 900 $N -k regex:k_accel -o /tmp/ncu/k_accel_c1 python tools/prof_accel.py --cfg 1 --reps 1 >> gpurun_out/r2l/ncu_full.log 2>&1
timeout 900 $N -k regex:k_accel -o /tmp/ncu/k_accel_c4 python tools/prof_accel.py --cfg 4 --reps 1 >> gpurun_out/r2l/ncu_full.log 2>&1
timeout 900 $N -k regex:k_accel -o /tmp/ncu/k_accel_c2 python tools/prof_accel.py --cfg 2 --reps 1 >> gpurun_out/r2l/ncu_full.log 2>&1
cp profiles/ncu_summary.json gpurun_out/r2l/
NCU_SUMMARY_DIR=gpurun_out/r2l python tools/ncu_summary.py k_accel_c3=/tmp/ncu/k_accel_c3.ncu-rep@k_accel \
  k_accel_c1=/tmp/ncu/k_accel_c1.ncu-rep@k_accel k_accel_c4=/tmp/ncu/k_accel_c4.ncu-rep@k_accel \
  k_accel_c2=/tmp/ncu/k_accel_c2.ncu-rep@k_accel > /dev/null
ncu -i /tmp/ncu/k_accel_c3.ncu-rep --page source --csv --print-source sass > gpurun_out/r2l/k_accel_c3_sass.csv 2>/dev/null
ncu -i /tmp/ncu/k_accel_c3.ncu-rep --page details --csv > gpurun_out/r2l/k_accel_c3_details.csv 2>/dev/null
cp /tmp/ncu/k_accel_c3.ncu-rep gpurun_out/r2l/ 2>/dev/null
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2l/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r2l/ncu_launch.log 2>&1
du -sh gpurun_out
tail -3 gpurun_out/r2l/pytest_gpu.log
