// setup.cuh -- per-bin setup (build_noise_scm / init_params) and the slot
// precompute stream kernel (sigma / tau) for the rcscm B200 path.
//
// Reference: model.hpp:58-124, linalg.hpp:25-86, ilrma.hpp:78-83,
//            solver_accel.hpp:33-64.
#pragma once

#include "common.cuh"

namespace rcscm {

// Device problem descriptor (device layout: bins flattened utterance-major,
// per-slot arrays [bin][t], X [bin][t][m]).
struct DevProblem {
  int64_t nb;        // total bins = B * I
  int64_t I;         // bins per utterance
  int64_t J;         // frames
  int M;             // mics
  int K;             // NMF rank (setup only)
  int n_h;           // target index
  const double2* X;  // [bin][t][m]
  const double2* W;  // [bin][M*M] col-major
  const double2* A;  // [bin][M*M] col-major
  const double* T;   // [u][i + k*I]
  const double* V;   // [u][k + t*K]
  // per-bin model inputs
  double2* a;    // [bin][M]
  double2* b;    // [bin][M]
  double2* Rp;   // [bin][M*M]
  double2* Rpp;  // [bin][M*M]
  double* power;  // [bin][M] mean demixed powers (setup scratch)
  // precompute outputs
  double2* sigma_ab;  // [bin]
  double* tau_aa;     // [bin]
  double2* sigma_bx;  // [bin][t]
  double2* tau_ax;    // [bin][t]
  double* tau_xx;     // [bin][t]
  // parameters
  double* r_h;     // [bin][t]
  double* r_u;     // [bin][t]
  double* lambda;  // [bin]
  double* logpdet;  // [bin] log pseudo-determinant of R' (product of its M-1 largest eigenvalues)
  unsigned long long* err;
};

// ---------------------------------------------------------------------------
// Cyclic complex Jacobi eigensolver for one M x M Hermitian matrix held by one
// thread (stand-in for Eigen::SelfAdjointEigenSolver, linalg.hpp:25-34). The
// rotation J = diag(1, conj(e)) [[c, s], [-s, c]] on (p, q) zeroes H(p, q); sweeps
// stop when no |H(p, q)| exceeds 1e-18 ||H||_F. On exit vals[] are ascending and
// V's column k (V[r + k*M]) is the matching unit eigenvector. Same algorithm as
// the oracle's restatement.
template <int M>
__device__ bool hermitian_eig_jacobi(double2 (&H)[M * M], double (&vals)[M], double2 (&V)[M * M]) {
  double fro = 0.0;
#pragma unroll
  for (int k = 0; k < M * M; ++k) fro += cnorm(H[k]);
  fro = sqrt(fro);
  if (!isfinite(fro)) return false;
  const double thresh = 1e-18 * fro;
#pragma unroll
  for (int c = 0; c < M; ++c) {
#pragma unroll
    for (int r = 0; r < M; ++r) V[r + c * M] = make_double2(r == c ? 1.0 : 0.0, 0.0);
    H[c + c * M].y = 0.0;
  }
  for (int sweep = 0; sweep < 100; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < M - 1; ++p) {
      for (int q = p + 1; q < M; ++q) {
        const double2 g = H[p + q * M];
        const double ag = sqrt(cnorm(g));
        if (!(ag > thresh)) continue;
        rotated = true;
        const double app = H[p + p * M].x, aqq = H[q + q * M].x;
        const double tau = (aqq - app) / (2.0 * ag);
        const double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        const double c = 1.0 / sqrt(1.0 + t * t);
        const double s = t * c;
        const double2 e = make_double2(g.x / ag, g.y / ag);
        const double2 eb = cconj(e);
        for (int k = 0; k < M; ++k) {  // H <- H J
          const double2 hkp = H[k + p * M], hkq = H[k + q * M];
          const double2 sebq = cmul(cscale(eb, s), hkq);
          const double2 cebq = cmul(cscale(eb, c), hkq);
          H[k + p * M] = csub(cscale(hkp, c), sebq);
          H[k + q * M] = cadd(cscale(hkp, s), cebq);
        }
        for (int k = 0; k < M; ++k) {  // H <- J^H H
          const double2 hpk = H[p + k * M], hqk = H[q + k * M];
          const double2 seq = cmul(cscale(e, s), hqk);
          const double2 ceq = cmul(cscale(e, c), hqk);
          H[p + k * M] = csub(cscale(hpk, c), seq);
          H[q + k * M] = cadd(cscale(hpk, s), ceq);
        }
        H[p + q * M] = make_double2(0.0, 0.0);
        H[q + p * M] = make_double2(0.0, 0.0);
        H[p + p * M] = make_double2(app - t * ag, 0.0);
        H[q + q * M] = make_double2(aqq + t * ag, 0.0);
        for (int k = 0; k < M; ++k) {  // V <- V J
          const double2 vkp = V[k + p * M], vkq = V[k + q * M];
          V[k + p * M] = csub(cscale(vkp, c), cmul(cscale(eb, s), vkq));
          V[k + q * M] = cadd(cscale(vkp, s), cmul(cscale(eb, c), vkq));
        }
      }
    }
    if (!rotated) break;
  }
  // Stable insertion sort by eigenvalue, permuting V's columns.
  int order[M];
#pragma unroll
  for (int k = 0; k < M; ++k) {
    order[k] = k;
    vals[k] = H[k + k * M].x;
  }
  for (int k = 1; k < M; ++k) {
    const int ok = order[k];
    const double vk = vals[k];
    int j = k - 1;
    while (j >= 0 && vals[j] > vk) {
      vals[j + 1] = vals[j];
      order[j + 1] = order[j];
      --j;
    }
    vals[j + 1] = vk;
    order[j + 1] = ok;
  }
  double2 Vs[M * M];
  for (int k = 0; k < M; ++k)
    for (int r = 0; r < M; ++r) Vs[r + k * M] = V[r + order[k] * M];
#pragma unroll
  for (int k = 0; k < M * M; ++k) V[k] = Vs[k];
  return true;
}

// ---------------------------------------------------------------------------
// K1a: mean demixed powers p_n = (1/J) sum_t |w_n^H x_t|^2, n != n_h
// (model.hpp:74-77). One CTA per bin, deterministic block reduction.
template <int M, int NT>
__global__ void __launch_bounds__(NT) k_setup_power(DevProblem P) {
  __shared__ double2 sW[M * M];
  __shared__ double red[M][NT / 32];
  const int64_t bin = blockIdx.x;
  const int tid = threadIdx.x;
  for (int k = tid; k < M * M; k += NT) sW[k] = P.W[bin * M * M + k];
  __syncthreads();
  double acc[M];
#pragma unroll
  for (int n = 0; n < M; ++n) acc[n] = 0.0;
  const double2* xb = P.X + bin * P.J * M;
  for (int64_t t = tid; t < P.J; t += NT) {
    double2 x[M];
#pragma unroll
    for (int m = 0; m < M; ++m) x[m] = xb[t * M + m];
#pragma unroll
    for (int n = 0; n < M; ++n) {
      double2 y = make_double2(0.0, 0.0);
#pragma unroll
      for (int m = 0; m < M; ++m) y = cfma(sW[n + m * M], x[m], y);
      acc[n] += cnorm(y);
    }
  }
  const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int n = 0; n < M; ++n) {
    const double s = warp_sum(acc[n]);
    if (lane == 0) red[n][warp] = s;
  }
  __syncthreads();
  if (tid < M) {
    double s = 0.0;
    for (int w = 0; w < NT / 32; ++w) s += red[tid][w];
    P.power[bin * M + tid] = (tid == P.n_h) ? 0.0 : s / static_cast<double>(P.J);
  }
}

// ---------------------------------------------------------------------------
// K1b: per-bin model setup, one thread per bin (model.hpp:58-90 build_noise_scm
// and the lambda rule of model.hpp:112-121). MODE 0: build R' from (A, power)
// and derive a, b, R'^+, lambda0. MODE 1: lambda0 only, from a given R'.
// MODE 2: log pseudo-determinant only (for the O(1) objective). Every mode
// writes logpdet when the pointer is set.
template <int M, int MODE>
__global__ void k_setup_bin(DevProblem P, double rank_tol, double eps) {
  const int64_t bin = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (bin >= P.nb) return;
  double2 H[M * M];
  if (MODE == 0) {
    double2 Am[M * M];
    double pw[M];
#pragma unroll
    for (int k = 0; k < M * M; ++k) Am[k] = P.A[bin * M * M + k];
#pragma unroll
    for (int n = 0; n < M; ++n) pw[n] = P.power[bin * M + n];
    double2 rp[M * M];
    for (int c = 0; c < M; ++c)
      for (int r = 0; r < M; ++r) {
        double2 s = make_double2(0.0, 0.0);
        for (int n = 0; n < M; ++n) {
          const double2 ap = cscale(Am[r + n * M], pw[n]);
          s = cadd(s, cmul(ap, cconj(Am[c + n * M])));
        }
        rp[r + c * M] = s;
      }
    for (int c = 0; c < M; ++c)
      for (int r = 0; r < M; ++r) {
        const double2 v = cadd(rp[r + c * M], cconj(rp[c + r * M]));
        H[r + c * M] = make_double2(v.x / 2.0, v.y / 2.0);
      }
    for (int k = 0; k < M * M; ++k) P.Rp[bin * M * M + k] = H[k];
    for (int r = 0; r < M; ++r) P.a[bin * M + r] = Am[r + P.n_h * M];
  } else {
    for (int k = 0; k < M * M; ++k) H[k] = P.Rp[bin * M * M + k];
  }
  double vals[M];
  double2 V[M * M];
  if (!hermitian_eig_jacobi<M>(H, vals, V)) {
    report_error(P.err, bin * P.J, kErrEigNoConverge);
    return;
  }
  const double lmax = std_max(vals[M - 1], 0.0);
  if (P.logpdet) {
    double lp = 0.0;
    for (int k = 1; k < M; ++k) lp += log(vals[k]);
    P.logpdet[bin] = lp;
  }
  if (MODE == 2) return;
  if (MODE == 0) {
    // null_eigenvector (linalg.hpp:74-86)
    const double cut_b = rank_tol * std_max(lmax, 1e-300);
    int near_zero = 0;
    for (int k = 0; k < M; ++k) near_zero += (vals[k] <= cut_b);
    if (near_zero != 1) {
      report_error(P.err, bin * P.J, kErrNullVector | (static_cast<unsigned>(min(near_zero, 15)) << 4));
      return;
    }
    // pseudo_inverse_psd (linalg.hpp:38-53)
    const double cut_p = rank_tol * lmax;
    if (vals[0] < -cut_p) {
      report_error(P.err, bin * P.J, kErrNotPsd);
      return;
    }
    // normalize_phase (linalg.hpp:58-70) of eigenvector 0
    double vmax = 0.0;
    for (int r = 0; r < M; ++r) vmax = fmax(vmax, sqrt(cnorm(V[r])));
    double2 f = make_double2(1.0, 0.0);
    if (vmax != 0.0) {
      int piv = 0;
      for (int r = 0; r < M; ++r)
        if (sqrt(cnorm(V[r])) > 1e-8 * vmax) {
          piv = r;
          break;
        }
      const double ap = sqrt(cnorm(V[piv]));
      f = make_double2(V[piv].x / ap, -V[piv].y / ap);
    }
    for (int r = 0; r < M; ++r) P.b[bin * M + r] = cmul(V[r], f);
    for (int c = 0; c < M; ++c)
      for (int r = 0; r < M; ++r) {
        double2 s = make_double2(0.0, 0.0);
        for (int k = 0; k < M; ++k) {
          if (vals[k] > cut_p) {
            const double inv = 1.0 / vals[k];
            s = cadd(s, cmul(cscale(V[r + k * M], inv), cconj(V[c + k * M])));
          }
        }
        P.Rpp[bin * M * M + r + c * M] = s;
      }
  }
  // init_params lambda0 (model.hpp:112-121), kDefaultRankTol cutoff.
  const double cut_l = 1e-10 * lmax;
  double lmin = vals[M - 1];
  for (int k = 0; k < M; ++k)
    if (vals[k] > cut_l) {
      lmin = vals[k];
      break;
    }
  P.lambda[bin] = std_max(lmin, eps);
}

// ---------------------------------------------------------------------------
// K1: slot stream kernel. One pass over x per slot:
//   INIT: r_h0 = max(sum_k T V, eps); r_u0 = max(Re(yh^H R'^+ yh)/M, eps),
//         yh = A (W x with entry n_h zeroed)          (model.hpp:102-111, ilrma.hpp:78-83)
//   PRE : sigma_bx = b^H x; tau_ax = (R'^+ a)^H x; tau_xx = max(Re(x^H R'^+ x), 0)
//         and per bin sigma_ab = a^H b, tau_aa = max(Re(a^H R'^+ a), 0)
//                                                    (solver_accel.hpp:33-64)
// Grid: (nb, ceil(J / NT)). HBM-bound: reads 16 M B/slot, writes <= 56 B/slot.
template <int M, int NT, bool INIT, bool PRE>
__global__ void __launch_bounds__(NT) k_slots(DevProblem P, double eps) {
  __shared__ double2 sRpp[M * M];
  __shared__ double2 sW[INIT ? M * M : 1];
  __shared__ double2 sA[INIT ? M * M : 1];
  __shared__ double2 sb[M];
  __shared__ double2 sp[M];  // R'^+ a
  const int64_t bin = blockIdx.x;
  const int tid = threadIdx.x;
  for (int k = tid; k < M * M; k += NT) {
    sRpp[k] = P.Rpp[bin * M * M + k];
    if (INIT) {
      sW[k] = P.W[bin * M * M + k];
      sA[k] = P.A[bin * M * M + k];
    }
  }
  if (PRE && tid < M) {
    sb[tid] = P.b[bin * M + tid];
    double2 s = make_double2(0.0, 0.0);
    for (int k = 0; k < M; ++k) s = cfma(P.Rpp[bin * M * M + tid + k * M], P.a[bin * M + k], s);
    sp[tid] = s;
  }
  __syncthreads();
  if (PRE && blockIdx.y == 0 && tid == 0) {
    double2 ab = make_double2(0.0, 0.0), aa = make_double2(0.0, 0.0);
    for (int k = 0; k < M; ++k) {
      const double2 ak = P.a[bin * M + k];
      ab = cfmac(ak, sb[k], ab);
      aa = cfmac(ak, sp[k], aa);
    }
    P.sigma_ab[bin] = ab;
    P.tau_aa[bin] = std_max(aa.x, 0.0);
  }
  const int64_t t = static_cast<int64_t>(blockIdx.y) * NT + tid;
  if (t >= P.J) return;
  const int64_t slot = bin * P.J + t;
  double2 x[M];
  const double2* xp = P.X + slot * M;
#pragma unroll
  for (int m = 0; m < M; ++m) x[m] = xp[m];
  if (PRE) {
    double2 sbx, tax;
    double txx;
    slot_forms<M>(x, sb, sp, sRpp, sbx, tax, txx);
    P.sigma_bx[slot] = sbx;
    P.tau_ax[slot] = tax;
    P.tau_xx[slot] = txx;
  }
  if (INIT) {
    double2 y[M];
#pragma unroll
    for (int n = 0; n < M; ++n) {
      double2 s = make_double2(0.0, 0.0);
#pragma unroll
      for (int m = 0; m < M; ++m) s = cfma(sW[n + m * M], x[m], s);
      y[n] = (n == P.n_h) ? make_double2(0.0, 0.0) : s;
    }
    double2 yh[M];
#pragma unroll
    for (int r = 0; r < M; ++r) {
      double2 s = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < M; ++k) s = cfma(sA[r + k * M], y[k], s);
      yh[r] = s;
    }
    double2 q = make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < M; ++r) {
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < M; ++k) acc = cfma(sRpp[r + k * M], yh[k], acc);
      q = cfmac(yh[r], acc, q);
    }
    P.r_u[slot] = std_max(q.x / M, eps);
    const int64_t u = bin / P.I, i = bin % P.I;
    const double* Tu = P.T + u * P.I * P.K;
    const double* Vu = P.V + u * P.K * P.J;
    double s = 0.0;
    for (int k = 0; k < P.K; ++k) s = fma(Tu[i + k * P.I], Vu[k + t * P.K], s);
    P.r_h[slot] = std_max(s, eps);
  }
}

}  // namespace rcscm

namespace rcscm {

// K1 (PRE): the per-slot quadratic forms of solver_accel.hpp:33-64 --
// sigma_bx = b^H x, tau_ax = (R'^+ a)^H x, tau_xx = max(Re x^H R'^+ x, 0) -- and
// the per-bin sigma_ab = a^H b, tau_aa = max(Re a^H R'^+ a, 0). One pass over x
// (16 M B/slot read, 40 B/slot written). Each thread owns SPT slots (strided by
// the CTA size, slot_grid) and issues all of its x loads before the per-bin
// prologue (R'^+, b, R'^+ a into shared memory), so the prologue's dependent
// loads and barrier overlap the stream instead of preceding it. Arithmetic order
// is that of k_slots (bitwise-identical results).
template <int M, int SPT>
__global__ void __launch_bounds__(256) k_pre(DevProblem P) {
  __shared__ double2 sRpp[M * M];
  __shared__ double2 sb[M];
  __shared__ double2 sp[M];  // R'^+ a
  const int64_t bin = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t J = P.J;
  const int64_t t0 = static_cast<int64_t>(blockIdx.y) * nt * SPT + tid;
  double2 x[SPT][M];
#pragma unroll
  for (int k = 0; k < SPT; ++k) {
    const int64_t t = t0 + static_cast<int64_t>(k) * nt;
    if (t < J) {
      const double2* xp = P.X + (bin * J + t) * M;
#pragma unroll
      for (int m = 0; m < M; ++m) x[k][m] = __ldg(xp + m);
    }
  }
  for (int k = tid; k < M * M; k += nt) sRpp[k] = P.Rpp[bin * M * M + k];
  if (tid < M) {
    sb[tid] = P.b[bin * M + tid];
    double2 s = make_double2(0.0, 0.0);
    for (int k = 0; k < M; ++k) s = cfma(P.Rpp[bin * M * M + tid + k * M], P.a[bin * M + k], s);
    sp[tid] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < SPT; ++k) {
    const int64_t t = t0 + static_cast<int64_t>(k) * nt;
    if (t >= J) continue;
    const int64_t slot = bin * J + t;
    double2 sbx, tax;
    double txx;
    slot_forms<M>(x[k], sb, sp, sRpp, sbx, tax, txx);
    P.sigma_bx[slot] = sbx;
    P.tau_ax[slot] = tax;
    P.tau_xx[slot] = txx;
  }
  if (blockIdx.y == 0 && tid == 0) {
    double2 ab = make_double2(0.0, 0.0), aa = make_double2(0.0, 0.0);
    for (int k = 0; k < M; ++k) {
      const double2 ak = P.a[bin * M + k];
      ab = cfmac(ak, sb[k], ab);
      aa = cfmac(ak, sp[k], aa);
    }
    P.sigma_ab[bin] = ab;
    P.tau_aa[bin] = std_max(aa.x, 0.0);
  }
}
// slots per thread of k_pre: 16 complex x values in registers
template <int M>
constexpr int pre_spt() {
  return M >= 16 ? 1 : 16 / M;
}

// K1 in the complex64 (FP32) mode: sigma_bx, tau_ax, tau_xx in single precision
// from the complex64 copy of x (solver_accel.hpp:33-64); the per-bin sigma_ab
// and tau_aa stay in double (computed from the double a, b, R'^+ exactly as
// k_slots does). Half the HBM bytes of the complex128 pass.
template <int M, int NT>
__global__ void __launch_bounds__(NT) k_slots_pre_f32(DevProblem P, const float2* __restrict__ Xf, float2* sbx_f,
                                                      float2* tax_f, float* txx_f) {
  __shared__ float2 sRpp[M * M];
  __shared__ float2 sb[M];
  __shared__ float2 sp[M];
  __shared__ double2 dp[M];
  const int64_t bin = blockIdx.x;
  const int tid = threadIdx.x;
  for (int k = tid; k < M * M; k += NT) sRpp[k] = to_c(P.Rpp[bin * M * M + k], 0.0f);
  if (tid < M) {
    sb[tid] = to_c(P.b[bin * M + tid], 0.0f);
    double2 s = make_double2(0.0, 0.0);
    for (int k = 0; k < M; ++k) s = cfma(P.Rpp[bin * M * M + tid + k * M], P.a[bin * M + k], s);
    dp[tid] = s;
    sp[tid] = to_c(s, 0.0f);
  }
  __syncthreads();
  if (blockIdx.y == 0 && tid == 0) {
    double2 ab = make_double2(0.0, 0.0), aa = make_double2(0.0, 0.0);
    for (int k = 0; k < M; ++k) {
      const double2 ak = P.a[bin * M + k];
      ab = cfmac(ak, P.b[bin * M + k], ab);
      aa = cfmac(ak, dp[k], aa);
    }
    P.sigma_ab[bin] = ab;
    P.tau_aa[bin] = std_max(aa.x, 0.0);
  }
  const int64_t t = static_cast<int64_t>(blockIdx.y) * NT + tid;
  if (t >= P.J) return;
  const int64_t slot = bin * P.J + t;
  float2 x[M];
#pragma unroll
  for (int m = 0; m < M; ++m) x[m] = Xf[slot * M + m];
  float2 sbx = make_float2(0.f, 0.f), tax = make_float2(0.f, 0.f), xx = make_float2(0.f, 0.f);
#pragma unroll
  for (int r = 0; r < M; ++r) {
    sbx = cfmac(sb[r], x[r], sbx);
    tax = cfmac(sp[r], x[r], tax);
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < M; ++k) acc = cfma(sRpp[r + k * M], x[k], acc);
    xx = cfmac(x[r], acc, xx);
  }
  sbx_f[slot] = sbx;
  tax_f[slot] = tax;
  txx_f[slot] = std_max(xx.x, 0.f);
}

// double <-> float element conversions (complex arrays pass 2 * count).
static __global__ void k_d2f(const double* __restrict__ src, float* __restrict__ dst, int64_t n) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[k] = static_cast<float>(src[k]);
}
static __global__ void k_f2d(const float* __restrict__ src, double* __restrict__ dst, int64_t n) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[k] = static_cast<double>(src[k]);
}

}  // namespace rcscm
