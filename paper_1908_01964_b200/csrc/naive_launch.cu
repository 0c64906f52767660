// naive_launch.cu -- launchers of K3 (naive.cuh) and K6 (accel1.cuh).
#include <cstdlib>

#include "dispatch.cuh"
#include "launch.h"

namespace rcscm {

#ifndef RCSCM_NAIVE_NT64_MIN_BINS
#define RCSCM_NAIVE_NT64_MIN_BINS 1480  // 64-thread CTAs from this many bins on (0: never)
#endif

// Threads stride over the bin's frames, so a CTA of NT threads runs ceil(J / NT)
// rounds and the last one may be partly idle: J = 320 takes 3 rounds of 128 (64
// lanes idle in the third, 20 % of the slot work) but exactly 5 rounds of 64, and
// 64-thread CTAs put five bins on an SM instead of two, so a bin's serial M-step
// (thread 0 inverts R_u) hides under other bins' slots. Once a batch fills the GPU
// with them (two waves of 148 x 5) the 64-thread kernel runs wherever it pads
// fewer frames; it emulates the 128-thread summation order (k_naive EMU), so every
// bit is the same and the choice may depend on the batch size (env
// RCSCM_NAIVE_NT64 = the fewest bins that take it, 0 disables it).
cudaError_t launch_naive(cudaStream_t s, int M, const NaiveArgs& N) {
  if (N.nb * N.J == 0) return cudaSuccess;
  const char* e = std::getenv("RCSCM_NAIVE_NT64");
  const int64_t min_nb = e ? std::atoll(e) : RCSCM_NAIVE_NT64_MIN_BINS;
  const int64_t pad128 = (N.J + 127) / 128 * 128, pad64 = (N.J + 63) / 64 * 64;
  const bool nt64 = min_nb > 0 && N.nb >= min_nb && pad64 < pad128;
  return dispatch_mics(M, [&](auto mm) {
    constexpr int MM = decltype(mm)::value;
    if (nt64) k_naive<MM, 64, true><<<N.nb, 64, 0, s>>>(N);
    else k_naive<MM, 128><<<N.nb, 128, 0, s>>>(N);
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
