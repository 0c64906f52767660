// accel_cl10.cu -- K2 instances for cluster size 10.
#include "accel_launch.cuh"

namespace rcscm {
cudaError_t launch_accel_cl10(cudaStream_t s, const AccelArgs& A, const AccelCfg& g) {
  return launch_accel_cl<10>(s, A, g);
}
}  // namespace rcscm
