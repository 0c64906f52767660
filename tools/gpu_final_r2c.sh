# round-2 final evidence on one B200: GPU suite, smoke, bench (both arms), the bench's
# ncu launch list (after the bench ran clean), ncu --set full of the naive kernel on C3 (32 utterances)
set -x
mkdir -p gpurun_out/final4 /tmp/ncu
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/final4/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final4/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final4/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final4/smoke.log
timeout 900 python bench.py > gpurun_out/final4/bench.json 2> gpurun_out/final4/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/final4/bench_ref.json 2> gpurun_out/final4/bench_ref.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/final4/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/final4/ncu_launch.log 2>&1
timeout 600 python tools/prof_accel.py --naive --cfg 3 --B 32 --reps 1 > gpurun_out/final4/naive_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -c 1 --launch-skip 3 -k regex:k_naive -o /tmp/ncu/k_naive_c3 python tools/prof_accel.py --naive --cfg 3 --B 32 --reps 1 > gpurun_out/final4/ncu_naive.log 2>&1
cp profiles/ncu_summary.json gpurun_out/final4/
NCU_SUMMARY_DIR=gpurun_out/final4 python tools/ncu_summary.py k_naive_c3=/tmp/ncu/k_naive_c3.ncu-rep@k_naive > /dev/null
tail -3 gpurun_out/final4/pytest_gpu.log; tail -2 gpurun_out/final4/smoke.log
