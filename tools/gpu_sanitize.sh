# compute-sanitizer, one tool at a time, on the small cases of tools/sanitize_cases.py
mkdir -p gpurun_out/sanitizer
CS="compute-sanitizer --print-limit 20 --error-exitcode 9"
for t in racecheck synccheck; do
  timeout 1500 $CS --tool $t python tools/sanitize_cases.py cluster2 cluster4 cluster16 single fused_c4 pipelined \
    > gpurun_out/sanitizer/$t.log 2>&1; echo "$t rc=$?" | tee -a gpurun_out/sanitizer/$t.log
done
timeout 1500 $CS --tool memcheck --leak-check full python tools/sanitize_cases.py > gpurun_out/sanitizer/memcheck.log 2>&1
echo "memcheck rc=$?" | tee -a gpurun_out/sanitizer/memcheck.log
timeout 900 $CS --tool initcheck python tools/sanitize_cases.py single pipelined naive_accel1 > gpurun_out/sanitizer/initcheck.log 2>&1
echo "initcheck rc=$?" | tee -a gpurun_out/sanitizer/initcheck.log
tail -3 gpurun_out/sanitizer/*.log
