# A/B builds of the library with extra -D flags: bash tools/ab_build.sh NAME "-DFOO=1 ..."
# -> build/ab/NAME/librcscm_gpu.so (select with RCSCM_GPU_LIB=...)
set -e
name=$1; shift
make -s -j10 -C paper_1908_01964_b200/csrc OUT=$PWD/build/ab/$name/librcscm_gpu.so OBJDIR=$PWD/build/ab/$name/obj \
  NVFLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr $*"
