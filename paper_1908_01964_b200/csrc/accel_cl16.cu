// accel_cl16.cu -- K2 instances for cluster size 16.
#include "accel_launch.cuh"

namespace rcscm {
cudaError_t launch_accel_cl16(cudaStream_t s, const AccelArgs& A, const AccelCfg& g) {
  return launch_accel_cl<16>(s, A, g);
}
}  // namespace rcscm
