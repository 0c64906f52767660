// accel_cl8.cu -- K2 instances for cluster size 8.
#include "accel_launch.cuh"

namespace rcscm {
cudaError_t launch_accel_cl8(cudaStream_t s, const AccelArgs& A, const AccelCfg& g) {
  return launch_accel_cl<8>(s, A, g);
}
}  // namespace rcscm
