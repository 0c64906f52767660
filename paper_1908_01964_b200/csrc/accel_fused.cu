// accel_fused.cu -- K2 instances with the sigma / tau precompute fused into the
// prologue (k_accel PREM = M), for the tuned single-CTA complex128 variant.
#include "accel_launch.cuh"

namespace rcscm {
#ifndef RCSCM_K2_W1_MINB
#define RCSCM_K2_W1_MINB 8  // one-warp CTAs per SM the launch bounds target (2 per SM sub-partition: 255 registers)
#endif
// one-warp CTAs (WE = 2: the 64 x 5 layout as 32 x 10), constants in registers
template <int PREM>
cudaError_t launch_w1(cudaStream_t s, const AccelArgs& A, const AccelCfg& g, bool epi) {
  if (g.we != 2 || g.spt != 10 || g.nt != 32) return cudaErrorInvalidValue;
  if (epi) return launch_accel_t<10, 1, true, false, 0, RCSCM_K2_W1_MINB, true, double, PREM, true, 2>(s, A, 32);
  return launch_accel_t<10, 1, true, false, 0, RCSCM_K2_W1_MINB, true, double, PREM, false, 2>(s, A, 32);
}

cudaError_t launch_accel_fused(cudaStream_t s, const AccelArgs& A, const AccelCfg& g) {
  const bool epi = A.dry_w || A.image_w;  // Wiener output as the epilogue (its own instantiation)
  if (g.we) {
    switch (g.prem) {
      case 2: return launch_w1<2>(s, A, g, epi);
      case 4: return launch_w1<4>(s, A, g, epi);
      case 8: return launch_w1<8>(s, A, g, epi);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (g.prem) {
    case 2:
      if (epi) return launch_accel_spt<1, true, false, 0, RCSCM_K2_MINB1, true, double, 2, true>(s, A, g.nt, g.spt);
      return launch_accel_spt<1, true, false, 0, RCSCM_K2_MINB1, true, double, 2>(s, A, g.nt, g.spt);
    case 4:
      if (epi) return launch_accel_spt<1, true, false, 0, RCSCM_K2_MINB1, true, double, 4, true>(s, A, g.nt, g.spt);
      return launch_accel_spt<1, true, false, 0, RCSCM_K2_MINB1, true, double, 4>(s, A, g.nt, g.spt);
    case 8:
      if (epi) return launch_accel_spt<1, true, false, 0, RCSCM_K2_MINB1, true, double, 8, true>(s, A, g.nt, g.spt);
      return launch_accel_spt<1, true, false, 0, RCSCM_K2_MINB1, true, double, 8>(s, A, g.nt, g.spt);
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace rcscm
