// accel_db_part.cu -- K2d instances with per-slot masks (ragged frame counts).
#include "accel_db_launch.cuh"

namespace rcscm {
cudaError_t launch_accel_db_part(cudaStream_t s, const AccelArgs& A, const AccelCfg& g) {
  return launch_db_m<false>(s, A, g);
}
}  // namespace rcscm
