# e2e run_algorithm2 wall time vs the chunk count and the number of output (D2H) segments
for ch in 4 8 16; do for s in 1 2 4 8 16; do
  [ $s -le $ch ] || continue
  echo "chunks=$ch segs=$s $(RCSCM_PIPELINE_CHUNKS=$ch RCSCM_D2H_SEGS=$s python tools/e2e_trace.py 2>&1 | grep 'wall per call')"
done; done
