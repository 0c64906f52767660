# e2e run_algorithm2 wall time vs the number of output (D2H) segments
for s in 1 2 4 8; do echo "segs=$s"; RCSCM_D2H_SEGS=$s python tools/e2e_trace.py 2>&1 | grep "wall per call"; done
