// accel_cl12.cu -- K2 instances for cluster size 12.
#include "accel_launch.cuh"

namespace rcscm {
cudaError_t launch_accel_cl12(cudaStream_t s, const AccelArgs& A, const AccelCfg& g) {
  return launch_accel_cl<12>(s, A, g);
}
}  // namespace rcscm
