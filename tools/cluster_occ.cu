// Co-resident clusters of the K2 cluster variants (cudaOccupancyMaxActiveClusters),
// i.e. how much of the GPU one launch of configs 2 / 4 can occupy at once.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_1908_01964_b200/csrc \
//        -o build/cluster_occ tools/cluster_occ.cu
#include <cstdio>

#include "accel.cuh"

using namespace rcscm;

template <int SPT, int CL, int SMEMC>
void report(const char* name, int nt) {
  auto kern = k_accel<SPT, CL, false, false, SMEMC, 0, true, double, 0>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL * 1024);
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = SMEMC ? static_cast<size_t>(SPT) * nt * (SMEMC == 1 ? 6 : 4) * sizeof(double) : 0;
  if (SMEMC) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.dynamicSmemBytes);
  if (CL > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.numAttrs = 1;
  cfg.attrs = attr;
  int n = -1;
  cudaError_t e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, kern);
  printf("%-28s CL=%2d nt=%3d SPT=%d smem=%zu regs=%d: max active clusters %d (%d CTAs of 148 SMs) %s\n", name, CL,
         nt, SPT, cfg.dynamicSmemBytes, fa.numRegs, n, n * CL, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  report<5, 16, 1>("config 2 (J=20000)", 256);
  report<5, 8, 1>("J=20000 as 8-CTA", 256);
  report<8, 2, 0>("config 4 (J=4096)", 256);
  report<4, 4, 1>("J=4096 as 4-CTA smem", 256);
  report<8, 4, 0>("J=4096 as 4-CTA x 128", 128);
  report<5, 2, 0>("J=640 as 2-CTA", 64);
  return 0;
}
