// ilrma.cu -- sphering and Gaussian ILRMA (iterative projection + NMF) on the GPU,
// the step before the SCM path, sm_100a.
//
// Reference: ilrma.hpp:53-73 (sphere), :100-123 (ilrma_nmf_update), :125-135
// (demixed_powers), :145-240 (run_ilrma). Layouts: X [bin][frame][mic];
// W, A [bin][M*M] column-major; T[n] I x K and V[n] K x J column-major (the
// reference's NmfModel); P[n] [bin][frame].
//
// Kernels (all reductions in a fixed order, so results are deterministic):
//   k_sphere       CTA per bin: covariance (lower triangle, block tree), one
//                  thread's Jacobi eig -> Q, then Q x for every frame
//   k_nmf_t        warp per (bin, source): R, P/R^2, 1/R on the fly, the K
//                  numerator / denominator sums over frames, T update
//   k_nmf_v        warp per (frame, source) over a transposed copy of P: the K
//                  sums over bins with the new T, V update
//   k_ip_cov       CTA per (bin, source): the weighted covariance U_n (lower
//                  triangle, block tree) -- independent of W, so all in parallel
//   k_ip_solve     thread per bin: the sequential row updates
//                  W_n <- (W U_n)^{-1} e_n / norm with Eigen::FullPivLU's pivot and
//                  rank rules (diagonal-loading retry)
//   k_powers       P[n] = |W x|^2 per slot + per-CTA partial sums for the mean
//   k_scale_mu     one CTA: mu_n = sqrt(mean P[n]) from the partials in order
//   k_scale_apply  W rows /= mu, P /= mu^2, T /= mu^2 (mu > 0 and finite)
//   k_demix_inv    thread per bin: A = W^{-1} (FullPivLU), singular -> error
#include "dispatch.cuh"
#include "launch.h"

namespace rcscm {

namespace {

constexpr double kNmfVarFloor = 1e-12;  // ilrma.hpp:40

// Eigen::FullPivLU on an M x M column-major matrix of one thread, in place in
// that thread's slice of shared memory (runtime loops: the row / column pivots
// index dynamically, which registers cannot). Pivot: first maximum |a_rc| in
// column-major order of the remaining corner; rank counts pivots above
// M * eps * |max pivot|. perm: 2M ints (row, then column transpositions).
template <int M>
struct DevFullPivLU {
  double2* lu;
  int* perm;
  int nonzero;
  double maxpivot;
  __device__ void compute() {
    nonzero = M;
    maxpivot = 0.0;
    for (int k = 0; k < M; ++k) {
      int br = k, bc = k;
      double big = -1.0;
      for (int c = k; c < M; ++c)
        for (int r = k; r < M; ++r) {
          const double v = cnorm(lu[r + c * M]);
          if (v > big) {
            big = v;
            br = r;
            bc = c;
          }
        }
      if (big == 0.0) {
        nonzero = k;
        for (int q = k; q < M; ++q) perm[q] = perm[M + q] = q;
        return;
      }
      maxpivot = fmax(maxpivot, sqrt(big));
      perm[k] = br;
      perm[M + k] = bc;
      if (br != k)
        for (int c = 0; c < M; ++c) {
          const double2 t = lu[k + c * M];
          lu[k + c * M] = lu[br + c * M];
          lu[br + c * M] = t;
        }
      if (bc != k)
        for (int r = 0; r < M; ++r) {
          const double2 t = lu[r + k * M];
          lu[r + k * M] = lu[r + bc * M];
          lu[r + bc * M] = t;
        }
      const double2 piv = lu[k + k * M];
      for (int r = k + 1; r < M; ++r) lu[r + k * M] = cdiv(lu[r + k * M], piv);
      for (int c = k + 1; c < M; ++c) {
        const double2 u = lu[k + c * M];
        for (int r = k + 1; r < M; ++r) lu[r + c * M] = csub(lu[r + c * M], cmul(lu[r + k * M], u));
      }
    }
  }
  __device__ bool invertible() const {
    const double thr = M * 2.220446049250313e-16 * maxpivot;
    int rk = 0;
    for (int q = 0; q < nonzero; ++q) rk += hypot(lu[q + q * M].x, lu[q + q * M].y) > thr;
    return rk == M;
  }
  // y := A^{-1} y
  __device__ void solve(double2* y) const {
    for (int k = 0; k < M; ++k) {
      const int r = perm[k];
      const double2 t = y[k];
      y[k] = y[r];
      y[r] = t;
    }
    for (int r = 0; r < M; ++r)
      for (int c = 0; c < r; ++c) y[r] = csub(y[r], cmul(lu[r + c * M], y[c]));
    for (int r = M - 1; r >= 0; --r) {
      for (int c = r + 1; c < M; ++c) y[r] = csub(y[r], cmul(lu[r + c * M], y[c]));
      y[r] = cdiv(y[r], lu[r + r * M]);
    }
    for (int k = M - 1; k >= 0; --k) {
      const int c = perm[M + k];
      const double2 t = y[k];
      y[k] = y[c];
      y[c] = t;
    }
  }
};
// threads per CTA of the thread-per-bin kernels (per-thread smem slices)
template <int M>
constexpr int lu_tpb() {
  return M <= 4 ? 32 : (M <= 8 ? 16 : 4);  // <= 48 KB of static shared memory
}
// per-thread shared slice: W, lu (M*M each), w (M) as double2 + 2M ints
template <int M>
constexpr int lu_slice() {
  return ((2 * M * M + M) * 16 + 2 * M * 4 + 15) / 16 * 16;  // 16-byte aligned slices
}

// Fixed-order block sum of NV doubles per thread (NT threads): xor butterfly in
// each warp, then the warp partials summed in warp order. out[NV] in shared
// memory; scratch red[NT/32][NV].
template <int NT, int NV>
__device__ void block_sum(const double (&v)[NV], double* red, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int e = 0; e < NV; ++e) {
    double s = v[e];
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
    if (lane == 0) red[warp * NV + e] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < NV; e += NT) {
    double s = 0.0;
    for (int w = 0; w < NT / 32; ++w) s += red[w * NV + e];
    out[e] = s;
  }
  __syncthreads();
}

}  // namespace

// ---- sphere (ilrma.hpp:53-73) ------------------------------------------------------
template <int M, int NT>
__global__ void __launch_bounds__(NT) k_sphere(const double2* __restrict__ X, int64_t J, double2* __restrict__ Q,
                                               double2* __restrict__ Xw) {
  constexpr int NE = M * (M + 1) / 2;  // lower triangle
  __shared__ double red[NT / 32 * 2 * NE];
  __shared__ double tot[2 * NE];
  __shared__ double2 sQ[M * M];
  const int64_t bin = blockIdx.x;
  double acc[2 * NE];
#pragma unroll
  for (int e = 0; e < 2 * NE; ++e) acc[e] = 0.0;
  for (int64_t t = threadIdx.x; t < J; t += NT) {
    double2 x[M];
#pragma unroll
    for (int m = 0; m < M; ++m) x[m] = X[(bin * J + t) * M + m];
    int e = 0;
#pragma unroll
    for (int c = 0; c < M; ++c)
#pragma unroll
      for (int r = c; r < M; ++r, ++e) {
        const double2 v = cmul(x[r], cconj(x[c]));
        acc[2 * e] += v.x;
        acc[2 * e + 1] += v.y;
      }
  }
  block_sum<NT, 2 * NE>(acc, red, tot);
  if (threadIdx.x == 0) {
    double2 H[M * M];
    int e = 0;
    for (int c = 0; c < M; ++c)
      for (int r = c; r < M; ++r, ++e) {
        const double2 v = make_double2(tot[2 * e] / static_cast<double>(J), tot[2 * e + 1] / static_cast<double>(J));
        H[r + c * M] = v;
        H[c + r * M] = cconj(v);
      }
    double tr = 0.0;
    for (int r = 0; r < M; ++r) tr += H[r + r * M].x;
    for (int r = 0; r < M; ++r) H[r + r * M].x += 1e-10 * tr / M;
    for (int r = 0; r < M; ++r) H[r + r * M].y = 0.0;  // (cov + cov^H) / 2
    double vals[M];
    double2 V[M * M];
    hermitian_eig_jacobi<M>(H, vals, V);
    for (int k = 0; k < M * M; ++k) sQ[k] = make_double2(0.0, 0.0);
    for (int k = 0; k < M; ++k) {
      const double s = 1.0 / sqrt(fmax(vals[k], 1e-300));
      for (int c = 0; c < M; ++c)
        for (int r = 0; r < M; ++r)
          sQ[r + c * M] = cadd(sQ[r + c * M], cscale(cmul(V[r + k * M], cconj(V[c + k * M])), s));
    }
    for (int k = 0; k < M * M; ++k) Q[bin * M * M + k] = sQ[k];
  }
  __syncthreads();
  for (int64_t t = threadIdx.x; t < J; t += NT) {
    double2 x[M];
#pragma unroll
    for (int m = 0; m < M; ++m) x[m] = X[(bin * J + t) * M + m];
#pragma unroll
    for (int r = 0; r < M; ++r) {
      double2 y = make_double2(0.0, 0.0);
#pragma unroll
      for (int c = 0; c < M; ++c) y = cfma(sQ[r + c * M], x[c], y);
      Xw[(bin * J + t) * M + r] = y;
    }
  }
}

// ---- NMF (ilrma.hpp:100-123) -----------------------------------------------------
// Warp reduce-scatter of 32 values per lane: after five halving steps (31
// shuffles instead of 32 x 5 for a butterfly per value) lane l holds the warp
// total of value l. Each partial sum is formed once, in a fixed order, so the
// result is deterministic.
__device__ __forceinline__ double warp_reduce_scatter32(const double (&v)[32]) {
  const int lane = threadIdx.x & 31;
  double a[16];
  {
    const bool up = lane & 16;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const double keep = up ? v[j + 16] : v[j], send = up ? v[j] : v[j + 16];
      a[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
  }
#pragma unroll
  for (int m = 8; m > 0; m >>= 1) {
    const bool up = lane & m;
#pragma unroll
    for (int j = 0; j < m; ++j) {
      const double keep = up ? a[j + m] : a[j], send = up ? a[j] : a[j + m];
      a[j] = keep + __shfl_xor_sync(0xffffffffu, send, m);
    }
  }
  return a[0];
}
// Warp totals of NV <= 32 values (zero-padded to 32): lane l gets the total of
// value l (0 for l >= NV).
template <int NV>
__device__ __forceinline__ double warp_totals(const double (&v)[NV]) {
  static_assert(NV <= 32, "at most 32 values");
  double w[32];
#pragma unroll
  for (int e = 0; e < 32; ++e) w[e] = e < NV ? v[e] : 0.0;
  return warp_reduce_scatter32(w);
}

// T update: one warp per (bin i, source n); lanes stride over frames, R = T V,
// P / R^2 and 1 / R on the fly, the K numerator / denominator sums over frames
// by a warp butterfly, lane k rewrites T(i, k).
template <int KMAX>
__global__ void __launch_bounds__(128) k_nmf_t(IlrmaArgs A, int M) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t I = A.I, J = A.J;
  const int K = A.K;
  if (w >= I * M) return;
  const int n = static_cast<int>(w / I);
  const int64_t i = w % I;
  double* T = A.T + static_cast<int64_t>(n) * I * K;
  const double* V = A.V + static_cast<int64_t>(n) * K * J;
  const double* P = A.P + (static_cast<int64_t>(n) * I + i) * J;
  double tk[KMAX], acc[2 * KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    tk[k] = k < K ? T[i + k * I] : 0.0;
    acc[2 * k] = acc[2 * k + 1] = 0.0;
  }
  for (int64_t t = lane; t < J; t += 32) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
      if (k < K) s = fma(tk[k], V[k + t * K], s);
    const double r = fmax(s, kNmfVarFloor);
    const double rinv = rcp_pos(r), pr2 = P[t] * rinv * rinv;  // MUFU + Newton, no IEEE divisions
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
      if (k < K) {
        const double v = V[k + t * K];
        acc[2 * k] = fma(pr2, v, acc[2 * k]);
        acc[2 * k + 1] = fma(rinv, v, acc[2 * k + 1]);
      }
  }
  // lane 2k: numerator total of base k; lane 2k + 1: its denominator (2 K <= 32)
  const double tot = warp_totals<2 * KMAX>(acc);
  const double den = __shfl_down_sync(0xffffffffu, tot, 1);
  const int k = lane >> 1;
  if (!(lane & 1) && k < K) T[i + k * I] = fmax(T[i + k * I] * sqrt(tot / fmax(den, 1e-300)), 1e-300);
}

// V update: one warp per (frame t, source n) over the transposed powers
// Pt[n][t][bin]; lanes stride over bins with the new T, lane k rewrites V(k, t).
template <int KMAX>
__global__ void __launch_bounds__(128) k_nmf_v(IlrmaArgs A, int M) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t I = A.I, J = A.J;
  const int K = A.K;
  if (w >= J * M) return;
  const int n = static_cast<int>(w / J);
  const int64_t t = w % J;
  const double* T = A.T + static_cast<int64_t>(n) * I * K;
  double* V = A.V + static_cast<int64_t>(n) * K * J;
  const double* Pt = A.Pt + (static_cast<int64_t>(n) * J + t) * I;
  double vk[KMAX], acc[2 * KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    vk[k] = k < K ? V[k + t * K] : 0.0;
    acc[2 * k] = acc[2 * k + 1] = 0.0;
  }
  for (int64_t i = lane; i < I; i += 32) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
      if (k < K) s = fma(T[i + k * I], vk[k], s);
    const double r = fmax(s, kNmfVarFloor);
    const double rinv = rcp_pos(r), pr2 = Pt[i] * rinv * rinv;
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
      if (k < K) {
        const double tv = T[i + k * I];
        acc[2 * k] = fma(tv, pr2, acc[2 * k]);
        acc[2 * k + 1] = fma(tv, rinv, acc[2 * k + 1]);
      }
  }
  const double tot = warp_totals<2 * KMAX>(acc);
  const double den = __shfl_down_sync(0xffffffffu, tot, 1);
  const int k = lane >> 1;
  if (!(lane & 1) && k < K) V[k + t * K] = fmax(V[k + t * K] * sqrt(tot / fmax(den, 1e-300)), 1e-300);
}

// ---- iterative projection (ilrma.hpp:190-216) -----------------------------------
// Pass 1: the weighted covariances U_n = (1/J) sum_t x x^H / r_n(t) do not depend
// on W, so all (bin, source) pairs run in parallel: CTA per (bin, source), lower
// triangle accumulated per thread, fixed-order block tree, full Hermitian U_n
// stored to ucov[(bin*M + n)][M*M].
template <int M, int NT>
__global__ void __launch_bounds__(NT) k_ip_cov(IlrmaArgs A) {
  constexpr int NE = M * (M + 1) / 2;
  __shared__ double red[NT / 32 * 2 * NE];
  __shared__ double tot[2 * NE];
  const int64_t i = blockIdx.x, I = A.I, J = A.J;
  const int n = blockIdx.y, K = A.K;
  const double* T = A.T + static_cast<int64_t>(n) * I * K;
  const double* V = A.V + static_cast<int64_t>(n) * K * J;
  double acc[2 * NE];
#pragma unroll
  for (int e = 0; e < 2 * NE; ++e) acc[e] = 0.0;
  for (int64_t t = threadIdx.x; t < J; t += NT) {
    double s = 0.0;
    for (int k = 0; k < K; ++k) s = fma(T[i + k * I], V[k + t * K], s);
    const double w = 1.0 / fmax(s, kNmfVarFloor);
    double2 x[M];
#pragma unroll
    for (int m = 0; m < M; ++m) x[m] = A.X[(i * J + t) * M + m];
    int e = 0;
#pragma unroll
    for (int c = 0; c < M; ++c)
#pragma unroll
      for (int r = c; r < M; ++r, ++e) {
        const double2 v = cscale(cmul(x[r], cconj(x[c])), w);
        acc[2 * e] += v.x;
        acc[2 * e + 1] += v.y;
      }
  }
  block_sum<NT, 2 * NE>(acc, red, tot);
  double2* U = A.ucov + (i * M + n) * M * M;
  for (int q = threadIdx.x; q < NE; q += NT) {
    int c = 0, r = q;  // q-th lower-triangle entry in (c, r >= c) order
    while (r >= M - c) {
      r -= M - c;
      ++c;
    }
    r += c;
    const double2 v = make_double2(tot[2 * q] / static_cast<double>(J), tot[2 * q + 1] / static_cast<double>(J));
    U[r + c * M] = v;
    U[c + r * M] = cconj(v);
  }
}

// Pass 1, warp form for M <= 5 (2 * NE <= 32): one warp per (bin, source),
// lanes stride over frames, the lower triangle reduced by a warp reduce-scatter.
template <int M>
__global__ void __launch_bounds__(128) k_ip_cov_warp(IlrmaArgs A) {
  constexpr int NE = M * (M + 1) / 2;
  static_assert(2 * NE <= 32, "warp form needs 2 NE <= 32");
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t I = A.I, J = A.J;
  const int K = A.K;
  if (w >= I * M) return;
  const int n = static_cast<int>(w % M);
  const int64_t i = w / M;
  const double* T = A.T + static_cast<int64_t>(n) * I * K;
  const double* V = A.V + static_cast<int64_t>(n) * K * J;
  double acc[2 * NE];
#pragma unroll
  for (int e = 0; e < 2 * NE; ++e) acc[e] = 0.0;
  for (int64_t t = lane; t < J; t += 32) {
    double s = 0.0;
    for (int k = 0; k < K; ++k) s = fma(T[i + k * I], V[k + t * K], s);
    const double wt = rcp_pos(fmax(s, kNmfVarFloor));
    double2 x[M];
#pragma unroll
    for (int m = 0; m < M; ++m) x[m] = A.X[(i * J + t) * M + m];
    int e = 0;
#pragma unroll
    for (int c = 0; c < M; ++c)
#pragma unroll
      for (int r = c; r < M; ++r, ++e) {
        const double2 v = cscale(cmul(x[r], cconj(x[c])), wt);
        acc[2 * e] += v.x;
        acc[2 * e + 1] += v.y;
      }
  }
  const double tot = warp_totals<2 * NE>(acc);  // lane 2q: Re of entry q, lane 2q + 1: Im
  const double im = __shfl_down_sync(0xffffffffu, tot, 1);
  if (!(lane & 1) && lane < 2 * NE) {
    int q = lane >> 1, c = 0;
    while (q >= M - c) {
      q -= M - c;
      ++c;
    }
    const int r = q + c;
    const double2 v = make_double2(tot / static_cast<double>(J), im / static_cast<double>(J));
    double2* U = A.ucov + (i * M + n) * M * M;
    U[r + c * M] = v;
    U[c + r * M] = cconj(v);
  }
}

// Pass 2: thread per bin, the sequential row updates (ilrma.hpp:195-215):
// W_n <- (W U_n)^{-1} e_n / sqrt(max(Re w^H U_n w, 1e-300)), conjugated into row n,
// with Eigen::FullPivLU's pivot / rank rules and the diagonal-loading retry.
// W, the LU and w live in the thread's shared-memory slice.
template <int M>
__global__ void __launch_bounds__(lu_tpb<M>()) k_ip_solve(IlrmaArgs A) {
  __shared__ __align__(16) unsigned char slab[lu_tpb<M>() * lu_slice<M>()];
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= A.I) return;
  double2* W = reinterpret_cast<double2*>(slab + threadIdx.x * lu_slice<M>());
  double2* lu = W + M * M;
  double2* w = lu + M * M;
  int* perm = reinterpret_cast<int*>(w + M);
  for (int k = 0; k < M * M; ++k) W[k] = A.W[i * M * M + k];
  DevFullPivLU<M> f{lu, perm, 0, 0.0};
  for (int n = 0; n < M; ++n) {
    const double2* U = A.ucov + (i * M + n) * M * M;
    auto form_wu = [&](double load) {  // lu = W U (+ load I)
      for (int c = 0; c < M; ++c)
        for (int r = 0; r < M; ++r) {
          double2 s = make_double2(0.0, 0.0);
          for (int k = 0; k < M; ++k) s = cfma(W[r + k * M], U[k + c * M], s);
          if (r == c) s.x += load;
          lu[r + c * M] = s;
        }
    };
    form_wu(0.0);
    double nrm = 0.0;
    for (int k = 0; k < M * M; ++k) nrm += cnorm(lu[k]);
    f.compute();
    bool ok = f.invertible();
    if (!ok) {  // diagonal-loading retry (ilrma.hpp:205-211)
      form_wu(1e-8 * fmax(sqrt(nrm), 1e-30));
      f.compute();
      ok = f.invertible();
    }
    if (!ok) {
      report_error(A.err, i * A.J, kErrIlrmaSpatial);
      return;  // the bin keeps its W (the reference stops updating it too)
    }
    for (int r = 0; r < M; ++r) w[r] = make_double2(r == n ? 1.0 : 0.0, 0.0);
    f.solve(w);
    double2 q = make_double2(0.0, 0.0);
    for (int r = 0; r < M; ++r) {
      double2 uw = make_double2(0.0, 0.0);
      for (int c = 0; c < M; ++c) uw = cfma(U[r + c * M], w[c], uw);
      q = cfmac(w[r], uw, q);
    }
    const double sc = sqrt(fmax(q.x, 1e-300));
    for (int c = 0; c < M; ++c) W[n + c * M] = cconj(make_double2(w[c].x / sc, w[c].y / sc));
  }
  for (int k = 0; k < M * M; ++k) A.W[i * M * M + k] = W[k];
}

// Pass 2, warp form for M <= 5: one warp per bin, lane l < M*M holding entry
// (l % M, l / M) -- column-major, so the lane index is Eigen's pivot tie-break
// order. The same FullPivLU pivot / rank rules and row updates as k_ip_solve,
// with the pivot search a warp (max |a|^2, min lane) reduction and the row /
// column swaps and eliminations lane shuffles.
__device__ __forceinline__ double2 shfl2(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}
template <int M>
__global__ void __launch_bounds__(128) k_ip_solve_warp(IlrmaArgs A) {
  static_assert(M * M <= 32, "warp form needs M*M <= 32");
  const int lane = threadIdx.x & 31;
  const int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  if (i >= A.I) return;
  const bool act = lane < M * M;
  const int r = lane % M, c = lane / M;
  double2 W = act ? A.W[i * M * M + lane] : make_double2(0.0, 0.0);
  for (int n = 0; n < M; ++n) {
    const double2 U = act ? A.ucov[(i * M + n) * M * M + lane] : make_double2(0.0, 0.0);
    // WU(r, c) = sum_k W(r, k) U(k, c)
    auto form_wu = [&](double load) {
      double2 s = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < M; ++k) {
        const double2 w = shfl2(W, act ? r + k * M : 0), u = shfl2(U, act ? k + c * M : 0);
        s = cfma(w, u, s);
      }
      if (r == c) s.x += load;
      return act ? s : make_double2(0.0, 0.0);
    };
    double2 a = form_wu(0.0);
    double nrm = cnorm(a);
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, m);
    int rowp[M], colp[M], nonzero = M;
    double maxpivot = 0.0;
    auto factor = [&]() {
      nonzero = M;
      maxpivot = 0.0;
      bool done = false;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        // pivot: max |a|^2 over the corner r, c >= k; ties -> lowest lane
        double v = (act && r >= k && c >= k && !done) ? cnorm(a) : -1.0;
        int l = lane;
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, v, m);
          const int ol = __shfl_xor_sync(0xffffffffu, l, m);
          if (ov > v || (ov == v && ol < l)) {
            v = ov;
            l = ol;
          }
        }
        if (!done && v == 0.0) {
          nonzero = k;
          done = true;
        }
        const int br = done ? k : l % M, bc = done ? k : l / M;
        rowp[k] = br;
        colp[k] = bc;
        if (done) continue;
        maxpivot = fmax(maxpivot, sqrt(v));
        // swap rows k and br, then columns k and bc
        int src = lane;
        if (r == k) src = br + c * M;
        else if (r == br) src = k + c * M;
        a = shfl2(a, act ? src : lane);
        src = lane;
        if (c == k) src = r + bc * M;
        else if (c == bc) src = r + k * M;
        a = shfl2(a, act ? src : lane);
        const double2 piv = shfl2(a, k + k * M);
        if (act && c == k && r > k) a = cdiv(a, piv);
        const double2 lrk = shfl2(a, act ? r + k * M : 0);  // L(r, k) after the division
        const double2 ukc = shfl2(a, act ? k + c * M : 0);  // U(k, c)
        if (act && r > k && c > k) a = csub(a, cmul(lrk, ukc));
      }
    };
    factor();
    const double thr = M * 2.220446049250313e-16 * maxpivot;
    auto rank_ok = [&]() {
      const bool big = act && r == c && r < nonzero && hypot(a.x, a.y) > thr;
      return __popc(__ballot_sync(0xffffffffu, big)) == M;
    };
    bool ok = rank_ok();
    if (!ok) {  // diagonal-loading retry (ilrma.hpp:205-211)
      a = form_wu(1e-8 * fmax(sqrt(nrm), 1e-30));
      factor();
      ok = rank_ok();
    }
    if (!ok) {
      if (lane == 0) report_error(A.err, i * A.J, kErrIlrmaSpatial);
      return;  // the bin keeps its W
    }
    // solve (W U) w = e_n with the factors: lanes 0..M-1 hold y
    double2 y = make_double2(lane == n ? 1.0 : 0.0, 0.0);
#pragma unroll
    for (int k = 0; k < M; ++k) {  // row transpositions
      const double2 yk = shfl2(y, k), yb = shfl2(y, rowp[k]);
      if (lane == k) y = yb;
      else if (lane == rowp[k]) y = yk;
    }
#pragma unroll
    for (int q = 0; q < M; ++q) {  // forward (unit lower)
      const double2 yq = shfl2(y, q);
      const double2 lrq = shfl2(a, lane < M ? lane + q * M : 0);
      if (lane > q && lane < M) y = csub(y, cmul(lrq, yq));
    }
#pragma unroll
    for (int q = M - 1; q >= 0; --q) {  // backward (upper)
      const double2 uqq = shfl2(a, q + q * M);
      if (lane == q) y = cdiv(y, uqq);
      const double2 yq = shfl2(y, q);
      const double2 urq = shfl2(a, lane < M ? lane + q * M : 0);
      if (lane < q) y = csub(y, cmul(urq, yq));
    }
#pragma unroll
    for (int k = M - 1; k >= 0; --k) {  // column transpositions
      const double2 yk = shfl2(y, k), yb = shfl2(y, colp[k]);
      if (lane == k) y = yb;
      else if (lane == colp[k]) y = yk;
    }
    // q = w^H U w; lane (r, c) forms U(r, c) w(c), rows summed in c order
    const double2 wc = shfl2(y, act ? c : 0);
    double2 t = act ? cmul(U, wc) : make_double2(0.0, 0.0);
    double2 uw = make_double2(0.0, 0.0);
#pragma unroll
    for (int cc = 0; cc < M; ++cc) uw = cadd(uw, shfl2(t, act ? r + cc * M : 0));  // lane (r, *): (U w)_r
    double2 qv = make_double2(0.0, 0.0);
#pragma unroll
    for (int rr = 0; rr < M; ++rr) qv = cfmac(shfl2(y, rr), shfl2(uw, rr), qv);
    const double sc = sqrt(fmax(qv.x, 1e-300));
    if (act && r == n) W = cconj(make_double2(wc.x / sc, wc.y / sc));
  }
  if (act) A.W[i * M * M + lane] = W;
}

// ---- demixed powers, scale normalisation, final inverse --------------------------
// P[n][i][t] = |(W_i x_it)_n|^2; partial[n][cta] = this CTA's sum (grid: bins x chunks)
template <int M, int NT>
__global__ void __launch_bounds__(NT) k_powers(IlrmaArgs A) {
  __shared__ double red[NT / 32 * M];
  __shared__ double tot[M];
  __shared__ double2 sW[M * M];
  const int64_t i = blockIdx.x, I = A.I, J = A.J;
  if (threadIdx.x < M * M) sW[threadIdx.x] = A.W[i * M * M + threadIdx.x];
  __syncthreads();
  double acc[M];
#pragma unroll
  for (int n = 0; n < M; ++n) acc[n] = 0.0;
  const int64_t t = static_cast<int64_t>(blockIdx.y) * NT + threadIdx.x;
  if (t < J) {
    double2 x[M];
#pragma unroll
    for (int m = 0; m < M; ++m) x[m] = A.X[(i * J + t) * M + m];
#pragma unroll
    for (int n = 0; n < M; ++n) {
      double2 y = make_double2(0.0, 0.0);
#pragma unroll
      for (int c = 0; c < M; ++c) y = cfma(sW[n + c * M], x[c], y);
      const double p = cnorm(y);
      A.P[(static_cast<int64_t>(n) * I + i) * J + t] = p;
      A.Pt[(static_cast<int64_t>(n) * J + t) * I + i] = p;
      acc[n] = p;
    }
  }
  block_sum<NT, M>(acc, red, tot);
  const int64_t cta = i * gridDim.y + blockIdx.y, ncta = I * gridDim.y;
  if (threadIdx.x < M) A.partial[threadIdx.x * ncta + cta] = tot[threadIdx.x];
}

// mu_n = sqrt(mean P[n]) (ilrma.hpp:221-229), partials summed in CTA order
__global__ void k_scale_mu(IlrmaArgs A, int64_t ncta, int M) {
  __shared__ double red[32 * 16];
  const int n = blockIdx.x;
  double s = 0.0;
  for (int64_t c = threadIdx.x; c < ncta; c += blockDim.x) s += A.partial[n * ncta + c];
  for (int m = 16; m > 0; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) tot += red[w];
    A.mu[n] = sqrt(tot / static_cast<double>(A.I * A.J));
  }
  (void)M;
}

// W rows /= mu, P /= mu^2, T /= mu^2 where mu > 0 and finite
__global__ void k_scale_apply(IlrmaArgs A, int M) {
  const int64_t I = A.I, J = A.J;
  const int K = A.K;
  const int64_t nP = static_cast<int64_t>(M) * I * J, nT = static_cast<int64_t>(M) * I * K,
                nW = I * static_cast<int64_t>(M) * M;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < nP + nT + nW;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int n;
    if (q < nP) {
      n = static_cast<int>(q / (I * J));
      const double mu = A.mu[n];
      if (mu > 0.0 && isfinite(mu)) {
        A.P[q] /= mu * mu;
        A.Pt[q] /= mu * mu;  // same source-major extent, transposed within
      }
    } else if (q < nP + nT) {
      const int64_t r = q - nP;
      n = static_cast<int>(r / (I * K));
      const double mu = A.mu[n];
      if (mu > 0.0 && isfinite(mu)) A.T[r] /= mu * mu;
    } else {
      const int64_t r = q - nP - nT;
      const int64_t e = r % (static_cast<int64_t>(M) * M);
      n = static_cast<int>(e % M);  // row of the column-major entry
      const double mu = A.mu[n];
      if (mu > 0.0 && isfinite(mu)) A.W[r] = make_double2(A.W[r].x / mu, A.W[r].y / mu);
    }
  }
}

// Inverse of the M x M matrix src (bin i) by the thread's shared-memory FullPivLU
// into dst; false if Eigen's rank rule calls it singular.
template <int M>
__device__ bool lu_inverse(unsigned char* slab, const double2* src, double2* dst) {
  double2* lu = reinterpret_cast<double2*>(slab + threadIdx.x * lu_slice<M>()) + M * M;
  double2* e = lu + M * M;
  int* perm = reinterpret_cast<int*>(e + M);
  for (int k = 0; k < M * M; ++k) lu[k] = src[k];
  DevFullPivLU<M> f{lu, perm, 0, 0.0};
  f.compute();
  if (!f.invertible()) return false;
  for (int c = 0; c < M; ++c) {
    for (int r = 0; r < M; ++r) e[r] = make_double2(r == c ? 1.0 : 0.0, 0.0);
    f.solve(e);
    for (int r = 0; r < M; ++r) dst[r + c * M] = e[r];
  }
  return true;
}

// A = W^{-1} per bin (ilrma.hpp:232-238)
template <int M>
__global__ void __launch_bounds__(lu_tpb<M>()) k_demix_inv(IlrmaArgs A) {
  __shared__ __align__(16) unsigned char slab[lu_tpb<M>() * lu_slice<M>()];
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= A.I) return;
  if (!lu_inverse<M>(slab, A.W + i * M * M, A.A + i * M * M)) report_error(A.err, i * A.J, kErrIlrmaDemix);
}

// ---- fold + target selection (tools/rcscm.cpp:173-181, model.hpp:43-54) -----------
// W_i = W_ilrma,i Q_i (back to the observation domain), A_i = W_i^{-1}
template <int M>
__global__ void __launch_bounds__(lu_tpb<M>()) k_fold(IlrmaArgs A, const double2* __restrict__ Q,
                                                     double2* __restrict__ Wout, double2* __restrict__ Aout) {
  __shared__ __align__(16) unsigned char slab[lu_tpb<M>() * lu_slice<M>()];
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= A.I) return;
  double2* W = reinterpret_cast<double2*>(slab + threadIdx.x * lu_slice<M>());
  for (int c = 0; c < M; ++c)
    for (int r = 0; r < M; ++r) {
      double2 s = make_double2(0.0, 0.0);
      for (int k = 0; k < M; ++k) s = cfma(A.W[i * M * M + r + k * M], Q[i * M * M + k + c * M], s);
      W[r + c * M] = s;
      Wout[i * M * M + r + c * M] = s;
    }
  if (!lu_inverse<M>(slab, W, Aout + i * M * M)) report_error(A.err, i * A.J, kErrIlrmaDemix);
}

// power[n][i] = ||(W_i X_i)_n||^2 ||A_i(:, n)||^2 (select_target_index, per bin)
template <int M, int NT>
__global__ void __launch_bounds__(NT) k_target_power(const double2* __restrict__ X, const double2* __restrict__ W,
                                                     const double2* __restrict__ Am, int64_t I, int64_t J,
                                                     double* __restrict__ power) {
  __shared__ double red[NT / 32 * M];
  __shared__ double tot[M];
  const int64_t i = blockIdx.x;
  double acc[M];
#pragma unroll
  for (int n = 0; n < M; ++n) acc[n] = 0.0;
  for (int64_t t = threadIdx.x; t < J; t += NT) {
    double2 x[M];
#pragma unroll
    for (int m = 0; m < M; ++m) x[m] = X[(i * J + t) * M + m];
#pragma unroll
    for (int n = 0; n < M; ++n) {
      double2 y = make_double2(0.0, 0.0);
#pragma unroll
      for (int c = 0; c < M; ++c) y = cfma(W[i * M * M + n + c * M], x[c], y);
      acc[n] += cnorm(y);
    }
  }
  block_sum<NT, M>(acc, red, tot);
  if (threadIdx.x < M) {
    const int n = threadIdx.x;
    double a2 = 0.0;
    for (int r = 0; r < M; ++r) a2 += cnorm(Am[i * M * M + r + n * M]);
    power[n * I + i] = tot[n] * a2;
  }
}

// ---- launchers -------------------------------------------------------------------
constexpr int kIlrmaNT = 128;

cudaError_t launch_sphere(cudaStream_t s, int M, const double2* X, int64_t I, int64_t J, double2* Q, double2* Xw) {
  if (I * J == 0) return cudaSuccess;
  return dispatch_mics(M, [&](auto mm) {
    constexpr int MM = decltype(mm)::value;
    k_sphere<MM, kIlrmaNT><<<static_cast<unsigned>(I), kIlrmaNT, 0, s>>>(X, J, Q, Xw);
    return cudaGetLastError();
  });
}

int64_t ilrma_partials(int64_t I, int64_t J) { return I * ((J + kIlrmaNT - 1) / kIlrmaNT); }

template <int KMAX>
static cudaError_t nmf_update(cudaStream_t s, const IlrmaArgs& A, int M) {
  k_nmf_t<KMAX><<<static_cast<unsigned>((A.I * M + 3) / 4), 128, 0, s>>>(A, M);
  k_nmf_v<KMAX><<<static_cast<unsigned>((A.J * M + 3) / 4), 128, 0, s>>>(A, M);
  return cudaGetLastError();
}

cudaError_t launch_ilrma_nmf(cudaStream_t s, const IlrmaArgs& A, int M) {
  if (A.K <= 4) return nmf_update<4>(s, A, M);
  if (A.K <= 8) return nmf_update<8>(s, A, M);
  if (A.K <= 16) return nmf_update<16>(s, A, M);
  return cudaErrorInvalidValue;
}

cudaError_t launch_ilrma_powers(cudaStream_t s, const IlrmaArgs& A, int M) {
  return dispatch_mics(M, [&](auto mm) {
    constexpr int MM = decltype(mm)::value;
    k_powers<MM, kIlrmaNT><<<dim3(static_cast<unsigned>(A.I), static_cast<unsigned>((A.J + kIlrmaNT - 1) / kIlrmaNT)),
                             kIlrmaNT, 0, s>>>(A);
    return cudaGetLastError();
  });
}

cudaError_t launch_ilrma_ip_scale(cudaStream_t s, const IlrmaArgs& A, int M) {
  cudaError_t e = dispatch_mics(M, [&](auto mm) {
    constexpr int MM = decltype(mm)::value;
    if constexpr (MM * (MM + 1) <= 32)
      k_ip_cov_warp<MM><<<static_cast<unsigned>((A.I * MM + 3) / 4), 128, 0, s>>>(A);
    else
      k_ip_cov<MM, kIlrmaNT><<<dim3(static_cast<unsigned>(A.I), MM), kIlrmaNT, 0, s>>>(A);
    if constexpr (MM * MM <= 32) {
      k_ip_solve_warp<MM><<<static_cast<unsigned>((A.I + 3) / 4), 128, 0, s>>>(A);
    } else {
      constexpr int tpb = lu_tpb<MM>();
      k_ip_solve<MM><<<static_cast<unsigned>((A.I + tpb - 1) / tpb), tpb, 0, s>>>(A);
    }
    return cudaGetLastError();
  });
  if (e != cudaSuccess) return e;
  if ((e = launch_ilrma_powers(s, A, M)) != cudaSuccess) return e;
  k_scale_mu<<<M, 512, 0, s>>>(A, ilrma_partials(A.I, A.J), M);
  k_scale_apply<<<148 * 8, 256, 0, s>>>(A, M);
  return cudaGetLastError();
}

cudaError_t launch_ilrma_fold(cudaStream_t s, const IlrmaArgs& A, int M, const double2* Q, double2* W, double2* Am) {
  return dispatch_mics(M, [&](auto mm) {
    constexpr int MM = decltype(mm)::value;
    constexpr int tpb = lu_tpb<MM>();
    k_fold<MM><<<static_cast<unsigned>((A.I + tpb - 1) / tpb), tpb, 0, s>>>(A, Q, W, Am);
    return cudaGetLastError();
  });
}

cudaError_t launch_target_power(cudaStream_t s, int M, const double2* X, const double2* W, const double2* Am,
                                int64_t I, int64_t J, double* power) {
  return dispatch_mics(M, [&](auto mm) {
    constexpr int MM = decltype(mm)::value;
    k_target_power<MM, kIlrmaNT><<<static_cast<unsigned>(I), kIlrmaNT, 0, s>>>(X, W, Am, I, J, power);
    return cudaGetLastError();
  });
}

cudaError_t launch_ilrma_inverse(cudaStream_t s, const IlrmaArgs& A, int M) {
  return dispatch_mics(M, [&](auto mm) {
    constexpr int MM = decltype(mm)::value;
    constexpr int tpb = lu_tpb<MM>();
    k_demix_inv<MM><<<static_cast<unsigned>((A.I + tpb - 1) / tpb), tpb, 0, s>>>(A);
    return cudaGetLastError();
  });
}

}  // namespace rcscm
