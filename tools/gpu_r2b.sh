# truth-based GPU parity: the table and the new tests
timeout 900 python tools/truth_table.py > gpurun_out/truth_table.md 2> gpurun_out/truth_table.err; echo "table rc=$?"
timeout 900 python -m pytest tests/test_gpu_truth.py -x -q -s > gpurun_out/pytest_truth.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_truth.log
cat gpurun_out/truth_table.md
