// accel_stream.cu -- launcher of the HBM-streaming Algorithm 2 (accel_stream.cuh)
// for bins longer than the on-chip kernel holds.
#include "accel_stream.cuh"
#include "launch.h"

namespace rcscm {

int64_t accel_stream_chunks(int64_t J) { return (J + kStreamChunk - 1) / kStreamChunk; }

cudaError_t launch_accel_stream(cudaStream_t s, const AccelArgs& A, double* partial, double* lam_buf, int* n_launch) {
  *n_launch = 0;
  if (A.nb * A.J == 0 || A.iters <= 0) return cudaSuccess;
  StreamAccelArgs P{};
  P.nb = A.nb;
  P.J = A.J;
  P.chunks = accel_stream_chunks(A.J);
  P.iters = A.iters;
  P.inv_M = A.inv_M;
  P.k1 = A.k1;
  P.k2 = A.k2;
  P.eps = A.eps;
  P.gamma_fault = A.gamma_fault;
  P.sigma_ab = A.sigma_ab;
  P.tau_aa = A.tau_aa;
  P.sigma_bx = A.sigma_bx;
  P.tau_ax = A.tau_ax;
  P.tau_xx = A.tau_xx;
  P.r_h = A.r_h;
  P.r_u = A.r_u;
  P.partial = partial;
  // lam_buf: [2][nb] lambda and [2][nb] its reciprocal, ping-pong by iteration;
  // the current lambda is never the array being written
  double* lam[2] = {lam_buf, lam_buf + A.nb};
  double* il[2] = {lam_buf + 2 * A.nb, lam_buf + 3 * A.nb};
  const dim3 grid(static_cast<unsigned>(A.nb), static_cast<unsigned>(P.chunks));
  for (int it = 0; it < A.iters; ++it) {
    P.it = it;
    P.r_h_in = it == 0 ? A.r_h_in : A.r_h;
    P.r_u_in = it == 0 ? A.r_u_in : A.r_u;
    P.lam_old = it == 0 ? A.lambda_in : lam[(it - 1) & 1];
    P.il_old = it == 0 ? nullptr : il[(it - 1) & 1];
    P.lam_new = lam[it & 1];
    P.il_new = il[it & 1];
    P.traj_r_h = A.traj_r_h;
    P.traj_r_u = A.traj_r_u;
    P.traj_lambda = A.traj_lambda;
    k_stream_term<<<grid, kStreamNT, 0, s>>>(P);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_stream_update<<<grid, kStreamNT, 0, s>>>(P);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    *n_launch += 2;
  }
  return cudaMemcpyAsync(A.lambda, lam[(A.iters - 1) & 1], A.nb * sizeof(double), cudaMemcpyDeviceToDevice, s);
}

}  // namespace rcscm
