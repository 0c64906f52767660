// naive_launch.cu -- launchers of K3 (naive.cuh) and K6 (accel1.cuh).
#include "dispatch.cuh"
#include "launch.h"

namespace rcscm {

constexpr int kNaiveNT = 128;

cudaError_t launch_naive(cudaStream_t s, int M, const NaiveArgs& N) {
  if (N.nb * N.J == 0) return cudaSuccess;
  return dispatch_mics(M, [&](auto mm) {
    constexpr int MM = decltype(mm)::value;
    k_naive<MM, kNaiveNT><<<N.nb, kNaiveNT, 0, s>>>(N);
    return cudaGetLastError();
  });
}

constexpr int kAccel1NT = 128;

cudaError_t launch_accel1(cudaStream_t s, int M, const Accel1Args& A) {
  if (A.nb * A.J == 0) return cudaSuccess;
  return dispatch_mics(M, [&](auto mm) {
    constexpr int MM = decltype(mm)::value;
    k_accel1<MM, kAccel1NT><<<A.nb, kAccel1NT, 0, s>>>(A);
    return cudaGetLastError();
  });
}

}  // namespace rcscm
