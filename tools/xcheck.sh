# protocol self-check: the NaN-poisoning build against the normal build, bitwise
python tools/xcheck.py gpurun_out/xcheck_normal.npz && \
RCSCM_GPU_LIB=$PWD/build/ab/xcheck/librcscm_gpu.so python tools/xcheck.py gpurun_out/xcheck_poison.npz && \
python tools/xcheck.py --compare gpurun_out/xcheck_normal.npz gpurun_out/xcheck_poison.npz
echo "xcheck rc=$?"
rm -f gpurun_out/xcheck_*.npz
