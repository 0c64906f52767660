// accel_fused.cu -- K2 instances with the sigma / tau precompute fused into the
// prologue (k_accel PREM = M), for the tuned single-CTA complex128 variant.
#include "accel_launch.cuh"

namespace rcscm {
cudaError_t launch_accel_fused(cudaStream_t s, const AccelArgs& A, const AccelCfg& g) {
  const bool epi = A.dry_w || A.image_w;  // Wiener output as the epilogue (its own instantiation)
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
