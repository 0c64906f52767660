// naive_launch.cu -- launcher of K3 (naive.cuh).
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

}  // namespace rcscm
