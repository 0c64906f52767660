// accel_db_launch.cuh -- launcher of K2d (accel_db.cuh) for one FULL flavour
// (instantiated by accel_db_full.cu / accel_db_part.cu so they compile in parallel).
#pragma once

#include "accel_db.cuh"
#include "launch.h"

namespace rcscm {

template <int CL, bool FULL, int PREM>
cudaError_t launch_db_t(cudaStream_t s, const AccelArgs& A, int nt) {
  auto kern = k_accel_db<CL, FULL, PREM>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>((A.nb + 1) / 2 * CL));
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  if (CL > 8) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, A);
}

template <bool FULL, int PREM>
cudaError_t launch_db_cl(cudaStream_t s, const AccelArgs& A, const AccelCfg& g) {
  switch (g.db_cl) {
    case 2: return launch_db_t<2, FULL, PREM>(s, A, g.db_nt);
    case 4: return launch_db_t<4, FULL, PREM>(s, A, g.db_nt);
    case 8: return launch_db_t<8, FULL, PREM>(s, A, g.db_nt);
    case 16: return launch_db_t<16, FULL, PREM>(s, A, g.db_nt);
    default: return cudaErrorInvalidValue;
  }
}

template <bool FULL>
cudaError_t launch_db_m(cudaStream_t s, const AccelArgs& A, const AccelCfg& g) {
  switch (g.prem) {
    case 2: return launch_db_cl<FULL, 2>(s, A, g);
    case 4: return launch_db_cl<FULL, 4>(s, A, g);
    case 8: return launch_db_cl<FULL, 8>(s, A, g);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_accel_db_full(cudaStream_t s, const AccelArgs& A, const AccelCfg& g);
cudaError_t launch_accel_db_part(cudaStream_t s, const AccelArgs& A, const AccelCfg& g);

}  // namespace rcscm
