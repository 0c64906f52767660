// accel_cl3.cu -- K2 instances for cluster size 3.
#include "accel_launch.cuh"

namespace rcscm {
cudaError_t launch_accel_cl3(cudaStream_t s, const AccelArgs& A, const AccelCfg& g) {
  return launch_accel_cl<3>(s, A, g);
}
}  // namespace rcscm
