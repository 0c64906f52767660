// accel_cl5.cu -- K2 instances for cluster size 5.
#include "accel_launch.cuh"

namespace rcscm {
cudaError_t launch_accel_cl5(cudaStream_t s, const AccelArgs& A, const AccelCfg& g) {
  return launch_accel_cl<5>(s, A, g);
}
}  // namespace rcscm
