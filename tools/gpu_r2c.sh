# truth parity + full-shape tests + K2 timing after the NaN-safe floor
timeout 900 python tools/truth_table.py > gpurun_out/truth_table.md 2> gpurun_out/truth_table.err; echo "table rc=$?"
timeout 1200 python -m pytest tests/test_gpu_truth.py tests/test_gpu_full.py -q -s > gpurun_out/pytest_truth.log 2>&1; echo "pytest rc=$?"
grep -E "accel2 c|naive c|C3 x8|passed|failed|Error" gpurun_out/pytest_truth.log | head -40
cat gpurun_out/truth_table.md
for a in "--cfg 1" "--cfg 3 --B 32" "--cfg 4" "--cfg 2"; do python tools/prof_accel.py $a --reps 5; done
