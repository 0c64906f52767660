// accel_fused.cu -- K2 instances with the sigma / tau precompute fused into the
// prologue (k_accel PREM = M), for the tuned single-CTA complex128 variant.
#include "accel_launch.cuh"

namespace rcscm {
cudaError_t launch_accel_fused(cudaStream_t s, const AccelArgs& A, const AccelCfg& g) {
  switch (g.prem) {
    case 2: return launch_accel_spt<1, true, false, 0, 3, true, double, 2>(s, A, g.nt, g.spt);
    case 4: return launch_accel_spt<1, true, false, 0, 3, true, double, 4>(s, A, g.nt, g.spt);
    case 8: return launch_accel_spt<1, true, false, 0, 3, true, double, 8>(s, A, g.nt, g.spt);
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace rcscm
