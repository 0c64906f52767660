# cluster-shape sweep of the current build (C4, C2): bash tools/gpu_cl_shapes.sh
for v in ":" "4:" "4:4" "3:"; do
  cl=${v%%:*}; spt=${v##*:}
  echo -n "C4 cl=$cl spt=$spt: "; RCSCM_ACCEL_CL=$cl RCSCM_ACCEL_SPT=$spt timeout 300 python tools/prof_accel.py --cfg 4 --reps 5 2>&1 | tail -1
done
for v in ":" "12:" "16:" "16:5"; do
  cl=${v%%:*}; spt=${v##*:}
  echo -n "C2 cl=$cl spt=$spt: "; RCSCM_ACCEL_CL=$cl RCSCM_ACCEL_SPT=$spt timeout 300 python tools/prof_accel.py --cfg 2 --reps 5 2>&1 | tail -1
done
