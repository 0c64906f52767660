# A/B builds of the library with extra -D flags:
#   bash tools/ab_build.sh NAME "-DFOO=1 ..." [obj.o ...]
# -> build/ab/NAME/librcscm_gpu.so (select with RCSCM_GPU_LIB=...). With object
# names given, the main build's objects are reused and only those are rebuilt
# with the flags (the rest keep the default flags).
set -e
name=$1; flags=$2; shift 2
obj=/tmp/ab_obj/$name
rm -rf $obj; mkdir -p $obj build/ab/$name
if [ $# -gt 0 ]; then
  cp build/csrc/*.o $obj/  # the main build's objects (build it first, from the main sources)
  for o in "$@"; do rm -f $obj/$o; done
fi
make -s -j10 -C paper_1908_01964_b200/csrc OUT=$PWD/build/ab/$name/librcscm_gpu.so OBJDIR=$obj \
  NVFLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr $flags"
