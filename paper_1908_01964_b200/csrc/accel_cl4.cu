// accel_cl4.cu -- K2 instances for cluster size 4.
#include "accel_launch.cuh"

namespace rcscm {
cudaError_t launch_accel_cl4(cudaStream_t s, const AccelArgs& A, const AccelCfg& g) {
  return launch_accel_cl<4>(s, A, g);
}
}  // namespace rcscm
