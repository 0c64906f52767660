#include <cstdlib>
// stream_launch.cu -- launchers of K4 (Wiener), the objective, the layout
// transposes and the FP64 probe (stream.cuh).
#include "dispatch.cuh"
#include "launch.h"

namespace rcscm {

constexpr int kWienerNT = 128;
constexpr int kObjNT = 128;

cudaError_t launch_wiener(cudaStream_t s, int M, const WienerArgs& W, bool from_x, bool noise) {
  if (W.nb * W.J == 0) return cudaSuccess;
  return dispatch_mics(M, [&](auto mm) {
    constexpr int MM = decltype(mm)::value;
    auto go = [&](auto kern, int spt) {
      const SlotGrid g = slot_grid(W.J, spt);
      kern<<<dim3(W.nb, g.chunks), g.nt, 0, s>>>(W);
      return cudaGetLastError();
    };
    if (from_x && noise) return go(k_wiener<MM, wiener_spt<MM, true>(), true, true>, wiener_spt<MM, true>());
    if (from_x) return go(k_wiener<MM, wiener_spt<MM, true>(), true, false>, wiener_spt<MM, true>());
    const char* e = std::getenv("RCSCM_STREAM_SPT");  // tuning knob
    const int spt = e ? std::atoi(e) : wiener_spt<MM, false>();
    if (spt == 1) return go(k_wiener<MM, 1, false, false>, 1);
    if (spt == 2) return go(k_wiener<MM, 2, false, false>, 2);
    return go(k_wiener<MM, wiener_spt<MM, false>(), false, false>, wiener_spt<MM, false>());
  });
}

cudaError_t launch_objective(cudaStream_t s, int M, ObjArgs O, int64_t* np) {
  dim3 grid(O.nb, (O.J + kObjNT - 1) / kObjNT);
  *np = static_cast<int64_t>(grid.x) * grid.y;
  if (O.nb * O.J == 0) return cudaSuccess;
  return dispatch_mics(M, [&](auto mm) {
    constexpr int MM = decltype(mm)::value;
    k_objective<MM, kObjNT><<<grid, kObjNT, 0, s>>>(O);
    return cudaGetLastError();
  });
}

cudaError_t launch_objective_fast(cudaStream_t s, ObjFastArgs O, int64_t* np) {
  dim3 grid(O.nb, (O.J + kObjNT - 1) / kObjNT);
  *np = static_cast<int64_t>(grid.x) * grid.y;
  if (O.nb * O.J == 0) return cudaSuccess;
  k_objective_fast<kObjNT><<<grid, kObjNT, 0, s>>>(O);
  return cudaGetLastError();
}

cudaError_t launch_sum_partials(cudaStream_t s, const double* partial, int64_t n, double* out) {
  k_sum_partials<<<1, 1024, 0, s>>>(partial, n, out);
  return cudaGetLastError();
}

cudaError_t launch_sum_rows(cudaStream_t s, const double* partial, int rows, int64_t n, double* out) {
  if (rows <= 0) return cudaSuccess;
  k_sum_rows<<<rows, 1024, 0, s>>>(partial, n, out);
  return cudaGetLastError();
}

template <class T, bool TO_BT>
static cudaError_t transpose(cudaStream_t s, const T* src, T* dst, int64_t B, int64_t I, int64_t J, int64_t ld) {
  if (B * I * J == 0) return cudaSuccess;
  dim3 grid((I + 31) / 32, (J + 31) / 32, B), block(32, 8);
  if (TO_BT)
    k_ij_to_bt<T><<<grid, block, 0, s>>>(src, dst, I, J, ld > 0 ? ld : I);
  else
    k_bt_to_ij<T><<<grid, block, 0, s>>>(src, dst, I, J, ld > 0 ? ld : I);
  return cudaGetLastError();
}

cudaError_t launch_to_bt(cudaStream_t s, const double* src, double* dst, int64_t B, int64_t I, int64_t J, int64_t ld) {
  return transpose<double, true>(s, src, dst, B, I, J, ld);
}
cudaError_t launch_to_ij(cudaStream_t s, const double* src, double* dst, int64_t B, int64_t I, int64_t J, int64_t ld) {
  return transpose<double, false>(s, src, dst, B, I, J, ld);
}
cudaError_t launch_to_ij_c(cudaStream_t s, const double2* src, double2* dst, int64_t B, int64_t I, int64_t J) {
  return transpose<double2, false>(s, src, dst, B, I, J, I);
}

cudaError_t launch_transpose_c(cudaStream_t s, const double2* src, double2* dst, int64_t I, int64_t J, int64_t ld,
                               bool to_bt) {
  return to_bt ? transpose<double2, true>(s, src, dst, 1, I, J, ld) : transpose<double2, false>(s, src, dst, 1, I, J, ld);
}

cudaError_t launch_fp64_probe(cudaStream_t s, int blocks, int iters, double* out) {
  k_fp64_probe<8><<<blocks, 256, 0, s>>>(1.0, iters, out);
  return cudaGetLastError();
}
cudaError_t launch_fp32_probe(cudaStream_t s, int blocks, int iters, double* out) {
  k_fp32_probe<8><<<blocks, 256, 0, s>>>(1.0f, iters, out);
  return cudaGetLastError();
}

cudaError_t launch_wiener_f32(cudaStream_t s, int M, const WienerArgsF32& W, bool from_x) {
  if (W.nb * W.J == 0) return cudaSuccess;
  return dispatch_mics(M, [&](auto mm) {
    constexpr int MM = decltype(mm)::value;
    dim3 grid(W.nb, (W.J + kWienerNT - 1) / kWienerNT);
    if (from_x)
      k_wiener_f32<MM, kWienerNT, true><<<grid, kWienerNT, 0, s>>>(W);
    else
      k_wiener_f32<MM, kWienerNT, false><<<grid, kWienerNT, 0, s>>>(W);
    return cudaGetLastError();
  });
}

}  // namespace rcscm
