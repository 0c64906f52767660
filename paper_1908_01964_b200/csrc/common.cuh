// common.cuh -- shared device helpers for the rcscm B200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace rcscm {

constexpr int kMaxMics = 16;

// std::max(v, lo) of the reference (returns v unless v < lo): a NaN v stays NaN,
// where fmax would replace it by lo and hide a non-finite input.
__device__ __forceinline__ double std_max(double v, double lo) { return v < lo ? lo : v; }
__device__ __forceinline__ float std_max(float v, float lo) { return v < lo ? lo : v; }

// Complex helpers on double2 (re, im).
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// conj(a) * b
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.x, b.y, -a.y * b.x));
}
// acc + a * b
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 acc) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, acc.x)), fma(a.x, b.y, fma(a.y, b.x, acc.y)));
}
// acc + conj(a) * b
__device__ __forceinline__ double2 cfmac(double2 a, double2 b, double2 acc) {
  return make_double2(fma(a.x, b.x, fma(a.y, b.y, acc.x)), fma(a.x, b.y, fma(-a.y, b.x, acc.y)));
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double cnorm(double2 a) { return fma(a.x, a.x, a.y * a.y); }
// a / b (Smith's algorithm: no overflow of |b|^2)
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  if (fabs(b.x) >= fabs(b.y)) {
    const double r = b.y / b.x, d = b.x + r * b.y;
    return make_double2((a.x + r * a.y) / d, (a.y - r * a.x) / d);
  }
  const double r = b.x / b.y, d = b.y + r * b.x;
  return make_double2((a.x * r + a.y) / d, (a.y * r - a.x) / d);
}

// The per-slot quadratic forms of solver_accel.hpp:33-64 for one x (M complex):
// sigma_bx = b^H x, tau_ax = (R'^+ a)^H x, tau_xx = max(Re x^H R'^+ x, 0), in
// the one arithmetic order shared by K1 (k_pre, k_slots) and K2's fused
// precompute, so both produce the same bits. tau_xx uses R'^+'s Hermitian
// symmetry (the reference evaluates the full form; rounding-level difference). sb = b, sp = R'^+ a, sR = R'^+
// (column-major M x M).
template <int M>
__device__ __forceinline__ void slot_forms(const double2 (&x)[M], const double2* sb, const double2* sp,
                                           const double2* sR, double2& sbx, double2& tax, double& txx) {
  sbx = make_double2(0.0, 0.0);
  tax = make_double2(0.0, 0.0);
#pragma unroll
  for (int r = 0; r < M; ++r) {
    sbx = cfmac(sb[r], x[r], sbx);
    tax = cfmac(sp[r], x[r], tax);
  }
  // x^H R x of the Hermitian R from its lower triangle:
  //   sum_r R_rr |x_r|^2 + 2 sum_{r > c} Re(conj(x_r) R_rc x_c)
  // (a third of the FP64 work of the full quadratic form)
  double d = 0.0, o = 0.0;
#pragma unroll
  for (int r = 0; r < M; ++r) {
    d = fma(sR[r + r * M].x, cnorm(x[r]), d);
#pragma unroll
    for (int c = 0; c < r; ++c) {
      const double2 y = cmul(sR[r + c * M], x[c]);
      o = fma(x[r].x, y.x, fma(x[r].y, y.y, o));
    }
  }
  txx = std_max(fma(2.0, o, d), 0.0);
}

// Launch shape of the slot-stream kernels (K1 precompute, K4 Wiener): each
// thread owns SPT slots of one bin strided by the CTA size, a CTA covers one
// chunk of a bin's frames. The chunk count is the fewest with <= 256 threads,
// and the CTA size the smallest warp multiple covering the chunk, so a bin of
// J frames wastes < 32 * SPT slots (J = 640, SPT = 4: one 160-thread CTA).
struct SlotGrid {
  int nt;
  int64_t chunks;
};
inline SlotGrid slot_grid(int64_t J, int spt) {
  const int64_t cap = static_cast<int64_t>(spt) * 256;
  const int64_t chunks = J > 0 ? (J + cap - 1) / cap : 1;
  const int64_t per = (J + chunks - 1) / chunks;
  const int64_t nt = ((per + spt - 1) / spt + 31) / 32 * 32;
  return SlotGrid{static_cast<int>(nt > 0 ? nt : 32), chunks};
}

// Reciprocal for strictly positive, normal x: MUFU.RCP64H seed refined by one
// Newton step plus the cubic term (error ~ e0^3, far below 1 ulp for the
// ~2^-22 seed). Replaces the IEEE division slow path in the on-chip loop.
__device__ __forceinline__ double rcp_pos(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

// ---- complex64 (FP32 mode) counterparts ----------------------------------------
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.x, b.y, -a.y * b.x));
}
__device__ __forceinline__ float2 cfmac(float2 a, float2 b, float2 acc) {
  return make_float2(fmaf(a.x, b.x, fmaf(a.y, b.y, acc.x)), fmaf(a.x, b.y, fmaf(-a.y, b.x, acc.y)));
}
__device__ __forceinline__ float2 cfma(float2 a, float2 b, float2 acc) {
  return make_float2(fmaf(a.x, b.x, fmaf(-a.y, b.y, acc.x)), fmaf(a.x, b.y, fmaf(a.y, b.x, acc.y)));
}
__device__ __forceinline__ float cnorm(float2 a) { return fmaf(a.x, a.x, a.y * a.y); }
// MUFU.RCP seed + one Newton step (~1 ulp in FP32) for strictly positive x.
__device__ __forceinline__ float rcp_pos(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return fmaf(r, fmaf(-x, r, 1.0f), r);
}
__device__ __forceinline__ float2 to_c(double2 v, float) { return make_float2(static_cast<float>(v.x), static_cast<float>(v.y)); }
__device__ __forceinline__ double2 to_c(double2 v, double) { return v; }
template <class T>
struct CplxOf;
template <>
struct CplxOf<double> {
  using type = double2;
};
template <>
struct CplxOf<float> {
  using type = float2;
};

// Device error word: the lowest failing (slot << 8 | code) wins (atomicMin),
// so the reported failure is the first in the reference's (bin, frame) order.
enum ErrCode : unsigned {
  kErrNone = 0,
  kErrEStepSingular = 1,   // solver_naive.hpp:207-209
  kErrMStepSingular = 2,   // solver_naive.hpp:366-367
  kErrNullVector = 3,      // linalg.hpp:82-84 via model.hpp:82-86 (count in bits 4..7)
  kErrNotPsd = 4,          // linalg.hpp:41-44 via model.hpp:82-86
  kErrObjectiveNotPd = 5,  // model.hpp:141-143
  kErrObjectiveNonFinite = 6,  // model.hpp:151-153
  kErrEigNoConverge = 7,   // linalg.hpp:31-32
  kErrFirstStageLambda = 8,    // solver_accel.hpp:90-92
  kErrFirstStageSingular = 9,  // solver_accel.hpp:95-97
  kErrIlrmaSpatial = 10,       // ilrma.hpp:212-216
  kErrIlrmaDemix = 11,         // ilrma.hpp:232-236
};
__device__ __forceinline__ void report_error(unsigned long long* err, long long slot, unsigned code) {
  atomicMin(err, (static_cast<unsigned long long>(slot) << 8) | code);
}

// Deterministic warp sum (xor butterfly: every lane ends with the same value).
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

}  // namespace rcscm
