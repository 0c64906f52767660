# K2 iteration-loop unroll factor A/B on the current kernel. Build the variants first
# (from paper_1908_01964_b200/csrc), e.g. for u in 1 3:
#   make -j10 OUT=/root/repo/build/u$u/librcscm_gpu.so OBJDIR=/root/repo/build/obj_u$u \
#     NVFLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
#     --expt-relaxed-constexpr -DRCSCM_K2_UNROLL=$u"
run() { for r in 1 2 3; do python tools/prof_accel.py --cfg 1 --reps 10; done; python tools/prof_accel.py --cfg 3 --B 32 --reps 5; python tools/prof_accel.py --cfg 4 --reps 3; }
echo "unroll 2 (default)"; run
cp paper_1908_01964_b200/librcscm_gpu.so /tmp/u2.so
for u in 1 3; do cp build/u$u/librcscm_gpu.so paper_1908_01964_b200/librcscm_gpu.so; echo "unroll $u"; run; done
cp /tmp/u2.so paper_1908_01964_b200/librcscm_gpu.so
