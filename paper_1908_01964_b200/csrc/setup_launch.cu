// setup_launch.cu -- launchers of K1a / K1b / K1 (setup.cuh).
#include "dispatch.cuh"
#include "launch.h"

namespace rcscm {

bool mics_supported(int M) { return (M >= 1 && M <= 8) || M == 16; }

constexpr int kSlotNT = 128;

cudaError_t launch_setup(cudaStream_t s, const DevProblem& P, double rank_tol, double eps) {
  if (P.nb == 0) return cudaSuccess;
  return dispatch_mics(P.M, [&](auto mm) {
    constexpr int MM = decltype(mm)::value;
    k_setup_power<MM, 256><<<P.nb, 256, 0, s>>>(P);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_setup_bin<MM, 0><<<(P.nb + 63) / 64, 64, 0, s>>>(P, rank_tol, eps);
    return cudaGetLastError();
  });
}

cudaError_t launch_lambda0(cudaStream_t s, const DevProblem& P, double eps) {
  if (P.nb == 0) return cudaSuccess;
  return dispatch_mics(P.M, [&](auto mm) {
    constexpr int MM = decltype(mm)::value;
    k_setup_bin<MM, 1><<<(P.nb + 63) / 64, 64, 0, s>>>(P, 1e-10, eps);
    return cudaGetLastError();
  });
}

cudaError_t launch_logpdet(cudaStream_t s, const DevProblem& P) {
  if (P.nb == 0) return cudaSuccess;
  return dispatch_mics(P.M, [&](auto mm) {
    constexpr int MM = decltype(mm)::value;
    k_setup_bin<MM, 2><<<(P.nb + 63) / 64, 64, 0, s>>>(P, 1e-10, 0.0);
    return cudaGetLastError();
  });
}

cudaError_t launch_slots(cudaStream_t s, const DevProblem& P, bool init, bool pre, double eps) {
  if (P.nb * P.J == 0 || !(init || pre)) return cudaSuccess;
  return dispatch_mics(P.M, [&](auto mm) {
    constexpr int MM = decltype(mm)::value;
    dim3 grid(P.nb, (P.J + kSlotNT - 1) / kSlotNT);
    if (init && pre)
      k_slots<MM, kSlotNT, true, true><<<grid, kSlotNT, 0, s>>>(P, eps);
    else if (init)
      k_slots<MM, kSlotNT, true, false><<<grid, kSlotNT, 0, s>>>(P, eps);
    else
      k_slots<MM, kSlotNT, false, true><<<grid, kSlotNT, 0, s>>>(P, eps);
    return cudaGetLastError();
  });
}

}  // namespace rcscm
