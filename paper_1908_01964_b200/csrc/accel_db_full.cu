// accel_db_full.cu -- K2d instances whose CTAs own exactly nt * 4 frames of each bin.
#include "accel_db_launch.cuh"

namespace rcscm {
cudaError_t launch_accel_db_full(cudaStream_t s, const AccelArgs& A, const AccelCfg& g) {
  return launch_db_m<true>(s, A, g);
}
}  // namespace rcscm
