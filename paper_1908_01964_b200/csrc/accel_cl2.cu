// accel_cl2.cu -- K2 instances for cluster size 2.
#include "accel_launch.cuh"

namespace rcscm {
cudaError_t launch_accel_cl2(cudaStream_t s, const AccelArgs& A, const AccelCfg& g) {
  return launch_accel_cl<2>(s, A, g);
}
}  // namespace rcscm
