# one-warp K2 layout vs the 64 x 5 CTA on C3 (128 utterances): bash tools/gpu_w1.sh
timeout 600 python -m pytest tests/test_gpu_w1.py -q -x 2>&1 | tail -2
for rep in 1 2; do
  for v in main:2048 main:0 w1m8:2048; do
    n=${v%%:*}; t=${v##*:}
    if [ "$n" = main ]; then lib=""; else lib=$PWD/build/ab/$n/librcscm_gpu.so; fi
    echo -n "$n W1=$t: "; RCSCM_GPU_LIB=$lib RCSCM_ACCEL_W1=$t timeout 300 python tools/prof_accel.py --cfg 3 --B 128 --reps 5 2>&1 | tail -1
  done
done
