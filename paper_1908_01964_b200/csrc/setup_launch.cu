#include <cstdlib>
// setup_launch.cu -- launchers of K1a / K1b / K1 (setup.cuh).
#include <algorithm>

#include "dispatch.cuh"
#include "launch.h"

namespace rcscm {

bool mics_supported(int M) { return M >= 1 && M <= kMaxMics; }

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
    if (!init) {  // the precompute pass alone (every solve): k_pre
      constexpr int SPT = pre_spt<MM>();
      const char* e = std::getenv("RCSCM_STREAM_SPT");  // tuning knob
      const int spt = e ? std::atoi(e) : SPT;
      auto go = [&](auto kern, int sp) {
        const SlotGrid g = slot_grid(P.J, sp);
        kern<<<dim3(P.nb, g.chunks), g.nt, 0, s>>>(P);
        return cudaGetLastError();
      };
      if (spt == 1) return go(k_pre<MM, 1>, 1);
      if (spt == 2 && SPT >= 2) return go(k_pre<MM, (SPT >= 2 ? 2 : 1)>, 2);
      return go(k_pre<MM, SPT>, SPT);
    }
    dim3 grid(P.nb, (P.J + kSlotNT - 1) / kSlotNT);
    if (init && pre)
      k_slots<MM, kSlotNT, true, true><<<grid, kSlotNT, 0, s>>>(P, eps);
    else
      k_slots<MM, kSlotNT, true, false><<<grid, kSlotNT, 0, s>>>(P, eps);
    return cudaGetLastError();
  });
}

cudaError_t launch_slots_pre_f32(cudaStream_t s, const DevProblem& P, const float2* Xf, float2* sbx, float2* tax,
                                 float* txx) {
  if (P.nb * P.J == 0) return cudaSuccess;
  return dispatch_mics(P.M, [&](auto mm) {
    constexpr int MM = decltype(mm)::value;
    dim3 grid(P.nb, (P.J + kSlotNT - 1) / kSlotNT);
    k_slots_pre_f32<MM, kSlotNT><<<grid, kSlotNT, 0, s>>>(P, Xf, sbx, tax, txx);
    return cudaGetLastError();
  });
}

static int conv_blocks(int64_t n) { return static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 16)); }

cudaError_t launch_d2f(cudaStream_t s, const double* src, float* dst, int64_t n) {
  if (n == 0) return cudaSuccess;
  k_d2f<<<conv_blocks(n), 256, 0, s>>>(src, dst, n);
  return cudaGetLastError();
}
cudaError_t launch_f2d(cudaStream_t s, const float* src, double* dst, int64_t n) {
  if (n == 0) return cudaSuccess;
  k_f2d<<<conv_blocks(n), 256, 0, s>>>(src, dst, n);
  return cudaGetLastError();
}

}  // namespace rcscm
