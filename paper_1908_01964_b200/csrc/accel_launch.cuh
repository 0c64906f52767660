// accel_launch.cuh -- K2 launcher for one cluster size (instantiated by the
// accel_cl*.cu translation units so the variants compile in parallel).
#pragma once

#include "launch.h"

namespace rcscm {

template <int SPT, int CL, bool FULL, bool TRAJ, int SMEMC, int MINB = 0, bool DIRECT = false,
          typename T = double, int PREM = 0, bool EPI = false, int WE = 0>
cudaError_t launch_accel_t(cudaStream_t s, const AccelArgs& A, int nt) {
  auto kern = k_accel<SPT, CL, FULL, TRAJ, SMEMC, MINB, DIRECT, T, PREM, EPI, WE>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(A.nb * CL));
  cfg.blockDim = dim3(nt);
  // shared planes: tax + (txx, dd) [+ cc for SMEMC 1], one complex each per slot
  // (the Wiener epilogue reads tax and cc back: all three planes)
  const int planes = (SMEMC == 1 || EPI) ? 6 : (SMEMC == 2 ? 4 : 0);
  cfg.dynamicSmemBytes = static_cast<size_t>(SPT) * nt * planes * sizeof(T);
  if (planes) {  // opt in to the full dynamic allowance (static + dynamic may pass 48 KB)
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(cfg.dynamicSmemBytes));
    if (e != cudaSuccess) return e;
  }
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  cfg.numAttrs = 0;
  if (CL > 1) {
    if (CL > 8) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.numAttrs = 1;
  }
  cfg.attrs = attr;
  return cudaLaunchKernelEx(&cfg, kern, A);
}

// Slots per thread: 1-6 and 8 for single-CTA bins; a cluster is only chosen
// once a bin exceeds the next smaller shape (jc > 768 frames per CTA), so its
// CTAs hold 4, 5, 6 or 8 slots per thread -- the others are not instantiated.
template <int CL, bool FULL, bool TRAJ, int SMEMC, int MINB = 0, bool DIRECT = false, typename T = double,
          int PREM = 0, bool EPI = false>
cudaError_t launch_accel_spt(cudaStream_t s, const AccelArgs& A, int nt, int spt) {
  switch (spt) {
    case 1:
      if constexpr (CL == 1) return launch_accel_t<1, CL, FULL, TRAJ, SMEMC, MINB, DIRECT, T, PREM, EPI>(s, A, nt);
      break;
    case 2:
      if constexpr (CL == 1) return launch_accel_t<2, CL, FULL, TRAJ, SMEMC, MINB, DIRECT, T, PREM, EPI>(s, A, nt);
      break;
    case 3:
      if constexpr (CL == 1) return launch_accel_t<3, CL, FULL, TRAJ, SMEMC, MINB, DIRECT, T, PREM, EPI>(s, A, nt);
      break;
    case 4: return launch_accel_t<4, CL, FULL, TRAJ, SMEMC, MINB, DIRECT, T, PREM, EPI>(s, A, nt);
    case 5: return launch_accel_t<5, CL, FULL, TRAJ, SMEMC, MINB, DIRECT, T, PREM, EPI>(s, A, nt);
    case 6: return launch_accel_t<6, CL, FULL, TRAJ, SMEMC, MINB, DIRECT, T, PREM, EPI>(s, A, nt);
    case 8: return launch_accel_t<8, CL, FULL, TRAJ, SMEMC, MINB, DIRECT, T, PREM, EPI>(s, A, nt);
    default: break;
  }
  return cudaErrorInvalidValue;
}

// Clusters with the sigma / tau precompute fused into the prologue (PREM = M),
// constants in registers, direct form.
template <int CL, int PREM>
cudaError_t launch_accel_fused_cl_m(cudaStream_t s, const AccelArgs& A, const AccelCfg& g) {
  const bool epi = A.dry_w || A.image_w;  // Wiener output as the epilogue
  if (g.full) {
    if (epi) return launch_accel_spt<CL, true, false, 0, 0, true, double, PREM, true>(s, A, g.nt, g.spt);
    return launch_accel_spt<CL, true, false, 0, 0, true, double, PREM>(s, A, g.nt, g.spt);
  }
  if (epi) return launch_accel_spt<CL, false, false, 0, 0, true, double, PREM, true>(s, A, g.nt, g.spt);
  return launch_accel_spt<CL, false, false, 0, 0, true, double, PREM>(s, A, g.nt, g.spt);
}

template <int CL>
cudaError_t launch_accel_cl(cudaStream_t s, const AccelArgs& A, const AccelCfg& g) {
  if constexpr (CL >= 2) {
    if (g.prem) {
      switch (g.prem) {
        case 2: return launch_accel_fused_cl_m<CL, 2>(s, A, g);
        case 4: return launch_accel_fused_cl_m<CL, 4>(s, A, g);
        case 8: return launch_accel_fused_cl_m<CL, 8>(s, A, g);
        default: return cudaErrorInvalidValue;
      }
    }
  }
  const bool traj = A.traj_r_h != nullptr || A.obj_part != nullptr;  // per-iteration recording
  if (g.f32) {  // complex64 mode: direct form; shared-memory constants for large clusters
    if constexpr (CL == 1) {
      if (g.full && g.minb && g.nt <= 128) return launch_accel_spt<CL, true, false, 0, 3, true, float>(s, A, g.nt, g.spt);
    }
    if constexpr (CL >= 8) {
      if (g.smem) {
        if (g.full) return launch_accel_spt<CL, true, false, 1, 0, true, float>(s, A, g.nt, g.spt);
        return launch_accel_spt<CL, false, false, 1, 0, true, float>(s, A, g.nt, g.spt);
      }
    }
    if (g.full) return launch_accel_spt<CL, true, false, 0, 0, true, float>(s, A, g.nt, g.spt);
    return launch_accel_spt<CL, false, false, 0, 0, true, float>(s, A, g.nt, g.spt);
  }
  if (traj) return launch_accel_spt<CL, false, true, 0>(s, A, g.nt, g.spt);
  if constexpr (CL == 1) {
    // 128-thread CTAs, several per SM: the tuned single-CTA-per-bin variants
    if (g.full && g.minb && g.nt <= 128 && g.direct) {
      if (g.smem == 2 && g.minb == 4) return launch_accel_spt<CL, true, false, 2, 4, true>(s, A, g.nt, g.spt);
      if (g.smem == 1 && g.minb == 4) return launch_accel_spt<CL, true, false, 1, 4, true>(s, A, g.nt, g.spt);
      if (g.smem == 2 && g.minb == 5) return launch_accel_spt<CL, true, false, 2, 5, true>(s, A, g.nt, g.spt);
      if (g.smem == 0) return launch_accel_spt<CL, true, false, 0, RCSCM_K2_MINB1, true>(s, A, g.nt, g.spt);
    }
  }
  if (g.direct) {  // r_u from rho(lambda_new) after the reduction (the faster form on B200)
    if (g.smem) {
      if (g.full) return launch_accel_spt<CL, true, false, 1, 0, true>(s, A, g.nt, g.spt);
      return launch_accel_spt<CL, false, false, 1, 0, true>(s, A, g.nt, g.spt);
    }
    if (g.full) return launch_accel_spt<CL, true, false, 0, 0, true>(s, A, g.nt, g.spt);
    return launch_accel_spt<CL, false, false, 0, 0, true>(s, A, g.nt, g.spt);
  }
  if constexpr (CL == 1) {  // the affine (non-DIRECT) form: single-CTA bins only (tuning knob)
    if (g.smem) {
      if (g.full) return launch_accel_spt<CL, true, false, 1>(s, A, g.nt, g.spt);
      return launch_accel_spt<CL, false, false, 1>(s, A, g.nt, g.spt);
    }
    if (g.full) return launch_accel_spt<CL, true, false, 0>(s, A, g.nt, g.spt);
    return launch_accel_spt<CL, false, false, 0>(s, A, g.nt, g.spt);
  }
  return cudaErrorInvalidValue;
}

#define RCSCM_DECLARE_ACCEL_CL(CL) \
  cudaError_t launch_accel_cl##CL(cudaStream_t s, const AccelArgs& A, const AccelCfg& g);
RCSCM_DECLARE_ACCEL_CL(1)
RCSCM_DECLARE_ACCEL_CL(2)
RCSCM_DECLARE_ACCEL_CL(3)
RCSCM_DECLARE_ACCEL_CL(4)
RCSCM_DECLARE_ACCEL_CL(5)
RCSCM_DECLARE_ACCEL_CL(6)
RCSCM_DECLARE_ACCEL_CL(8)
RCSCM_DECLARE_ACCEL_CL(10)
RCSCM_DECLARE_ACCEL_CL(12)
RCSCM_DECLARE_ACCEL_CL(16)
// the fused-precompute instances (accel_fused.cu)
cudaError_t launch_accel_fused(cudaStream_t s, const AccelArgs& A, const AccelCfg& g);

}  // namespace rcscm
