// accel_cl6.cu -- K2 instances for cluster size 6.
#include "accel_launch.cuh"

namespace rcscm {
cudaError_t launch_accel_cl6(cudaStream_t s, const AccelArgs& A, const AccelCfg& g) {
  return launch_accel_cl<6>(s, A, g);
}
}  // namespace rcscm
