// accel_cl1.cu -- K2 instances for cluster size 1.
#include "accel_launch.cuh"

namespace rcscm {
cudaError_t launch_accel_cl1(cudaStream_t s, const AccelArgs& A, const AccelCfg& g) {
  return launch_accel_cl<1>(s, A, g);
}
}  // namespace rcscm
