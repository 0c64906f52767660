// naive.cuh -- K3: the naive EM rule with an explicit per-slot M x M Hermitian
// inverse (the comparison path), sm_100a.
//
// Reference: solver_naive.hpp:153-246 (E-step per slot), :319-386 (fused
// per-bin E/M iteration), :412-450 (run_naive), and the closed-form Hermitian
// PD inverses of :46-146 (S = 2, 3, 4; LLT for other sizes).
//
// Per slot (one thread), with R~_u = R' + lambda~ b b^H:
//   R_x   = r~_h a a^H + r~_u R~_u ;  R_x^{-1} explicitly (closed form / Cholesky)
//   r^_h  = r~_h - r~_h^2 a^H R_x^{-1} a + |r~_h x^H R_x^{-1} a|^2
//   R^_u  = r~_u R~_u - r~_u^2 R~_u R_x^{-1} R~_u + r~_u^2 v v^H,  v = R~_u R_x^{-1} x
// The M-step consumes R^_u only through b^H R^_u b (lambda) and
// tr(R_u^{-1} R^_u) (r_u), so those contractions are formed directly from
// R_x^{-1} instead of materialising / storing the M x M matrix per slot:
//   q   = b^H R^_u b      = r~_u b^H w - r~_u^2 w^H R_x^{-1} w + r~_u^2 |w^H z|^2
//   T_a = tr(R~_u^{-1} R^_u) = r~_u M - r~_u^2 tr(R_x^{-1} R~_u) + r~_u^2 z^H R~_u z
//   T_b = u^H R^_u u      = r~_u u^H b - r~_u^2 b^H R_x^{-1} b + r~_u^2 |b^H z|^2
//   with z = R_x^{-1} x, w = R~_u b, u = R~_u^{-1} b (per bin).
// lambda = max((1/J) sum_t q / r~_u, eps)              (solver_naive.hpp:336-355)
// R_u = R' + lambda b b^H = R~_u + d b b^H, d = lambda - lambda~, so by
// Sherman-Morrison R_u^{-1} = R~_u^{-1} - d u u^H / (1 + d b^H u) and
//   r_u = max((T_a - d / (1 + d b^H u) T_b) / M, eps) = max(tr(R_u^{-1} R^_u)/M, eps)
//                                                      (solver_naive.hpp:357-385)
// Only R' and b enter (as in the reference); R'^+ is not used.
#pragma once

#include "common.cuh"

namespace rcscm {

// ---- Hermitian PD inverse ---------------------------------------------------
// Full M x M column-major in/out. Returns false if not positive definite.
template <int M>
__device__ __forceinline__ bool herm_pd_inverse(const double2 (&R)[M * M], double2 (&O)[M * M]) {
  if constexpr (M == 1) {
    const double a = R[0].x;
    if (!(a > 0.0)) return false;
    O[0] = make_double2(1.0 / a, 0.0);
    return true;
  } else if constexpr (M == 2) {  // solver_naive.hpp:50-61
    const double a = R[0].x, c = R[3].x;
    const double2 b = R[2];  // R(0, 1)
    const double det = a * c - cnorm(b);
    if (!(a > 0.0) || !(det > 0.0)) return false;
    const double id = 1.0 / det;
    O[0] = make_double2(c * id, 0.0);
    O[3] = make_double2(a * id, 0.0);
    O[2] = make_double2(-b.x * id, -b.y * id);
    O[1] = make_double2(-b.x * id, b.y * id);
    return true;
  } else if constexpr (M == 3) {  // solver_naive.hpp:62-84
    const double a = R[0].x, b = R[4].x, c = R[8].x;
    const double2 d = R[3], e = R[6], f = R[7];  // (0,1) (0,2) (1,2)
    const double m00 = b * c - cnorm(f);
    const double m11 = a * c - cnorm(e);
    const double m22 = a * b - cnorm(d);
    // det = Re(a m00 - d (conj(d) c - f conj(e)) + e (conj(d) conj(f) - b conj(e)))
    const double2 t1 = csub(cscale(cconj(d), c), cmul(f, cconj(e)));
    const double2 t2 = csub(cmul(cconj(d), cconj(f)), cscale(cconj(e), b));
    const double det = a * m00 - cmul(d, t1).x + cmul(e, t2).x;
    if (!(a > 0.0) || !(m22 > 0.0) || !(det > 0.0)) return false;
    const double id = 1.0 / det;
    O[0] = make_double2(m00 * id, 0.0);
    O[4] = make_double2(m11 * id, 0.0);
    O[8] = make_double2(m22 * id, 0.0);
    const double2 o01 = cscale(csub(cmul(e, cconj(f)), cscale(d, c)), id);
    const double2 o02 = cscale(csub(cmul(d, f), cscale(e, b)), id);
    const double2 o12 = cscale(csub(cmul(e, cconj(d)), cscale(f, a)), id);
    O[3] = o01;
    O[6] = o02;
    O[7] = o12;
    O[1] = cconj(o01);
    O[2] = cconj(o02);
    O[5] = cconj(o12);
    return true;
  } else if constexpr (M == 4) {  // solver_naive.hpp:85-144 (2x2 block Schur)
#define RR(r, c) R[(r) + (c) * 4]
    const double a00 = RR(0, 0).x, a11 = RR(1, 1).x;
    const double2 a01 = RR(0, 1);
    const double det_a = a00 * a11 - cnorm(a01);
    if (!(a00 > 0.0) || !(det_a > 0.0)) return false;
    const double ida = 1.0 / det_a;
    const double ai00 = a11 * ida, ai11 = a00 * ida;
    const double2 ai01 = make_double2(-a01.x * ida, -a01.y * ida), ai10 = cconj(ai01);
    const double2 t00 = cadd(cscale(RR(0, 2), ai00), cmul(ai01, RR(1, 2)));
    const double2 t01 = cadd(cscale(RR(0, 3), ai00), cmul(ai01, RR(1, 3)));
    const double2 t10 = cadd(cmul(ai10, RR(0, 2)), cscale(RR(1, 2), ai11));
    const double2 t11 = cadd(cmul(ai10, RR(0, 3)), cscale(RR(1, 3), ai11));
    const double sc00 = RR(2, 2).x - (cmulc(RR(0, 2), t00).x + cmulc(RR(1, 2), t10).x);
    const double sc11 = RR(3, 3).x - (cmulc(RR(0, 3), t01).x + cmulc(RR(1, 3), t11).x);
    const double2 sc01 = csub(csub(RR(2, 3), cmulc(RR(0, 2), t01)), cmulc(RR(1, 2), t11));
    const double det_s = sc00 * sc11 - cnorm(sc01);
    if (!(sc00 > 0.0) || !(det_s > 0.0)) return false;
    const double ids = 1.0 / det_s;
    const double si00 = sc11 * ids, si11 = sc00 * ids;
    const double2 si01 = make_double2(-sc01.x * ids, -sc01.y * ids), si10 = cconj(si01);
    const double2 u00 = cadd(cscale(t00, si00), cmul(t01, si10));
    const double2 u01 = cadd(cmul(t00, si01), cscale(t01, si11));
    const double2 u10 = cadd(cscale(t10, si00), cmul(t11, si10));
    const double2 u11 = cadd(cmul(t10, si01), cscale(t11, si11));
#undef RR
#define OO(r, c) O[(r) + (c) * 4]
    OO(0, 0) = make_double2(ai00 + (cmul(u00, cconj(t00)).x + cmul(u01, cconj(t01)).x), 0.0);
    OO(1, 1) = make_double2(ai11 + (cmul(u10, cconj(t10)).x + cmul(u11, cconj(t11)).x), 0.0);
    OO(0, 1) = cadd(cadd(ai01, cmul(u00, cconj(t10))), cmul(u01, cconj(t11)));
    OO(1, 0) = cconj(OO(0, 1));
    OO(0, 2) = make_double2(-u00.x, -u00.y);
    OO(0, 3) = make_double2(-u01.x, -u01.y);
    OO(1, 2) = make_double2(-u10.x, -u10.y);
    OO(1, 3) = make_double2(-u11.x, -u11.y);
    OO(2, 0) = cconj(OO(0, 2));
    OO(3, 0) = cconj(OO(0, 3));
    OO(2, 1) = cconj(OO(1, 2));
    OO(3, 1) = cconj(OO(1, 3));
    OO(2, 2) = make_double2(si00, 0.0);
    OO(3, 3) = make_double2(si11, 0.0);
    OO(2, 3) = si01;
    OO(3, 2) = si10;
#undef OO
    return true;
  } else {
    // Cholesky R = L L^H (lower triangle read, Eigen::LLT semantics:
    // fail when a pivot is not > 0), then R^{-1} = L^{-H} L^{-1}.
    double2 L[M * M];
#pragma unroll
    for (int k = 0; k < M * M; ++k) L[k] = make_double2(0.0, 0.0);
    double dinv[M];
#pragma unroll
    for (int k = 0; k < M; ++k) {
      double x = R[k + k * M].x;
#pragma unroll
      for (int j = 0; j < k; ++j) x -= cnorm(L[k + j * M]);
      if (x <= 0.0) return false;  // Eigen::LLT's pivot test
      const double lkk = sqrt(x);
      dinv[k] = 1.0 / lkk;
      L[k + k * M] = make_double2(lkk, 0.0);
#pragma unroll
      for (int i = k + 1; i < M; ++i) {
        double2 s = R[i + k * M];
#pragma unroll
        for (int j = 0; j < k; ++j) s = csub(s, cmul(L[i + j * M], cconj(L[k + j * M])));
        L[i + k * M] = cscale(s, dinv[k]);
      }
    }
    // Linv (lower) by forward substitution, stored in L's slots.
    double2 Li[M * M];
#pragma unroll
    for (int k = 0; k < M * M; ++k) Li[k] = make_double2(0.0, 0.0);
#pragma unroll
    for (int c = 0; c < M; ++c) {
      Li[c + c * M] = make_double2(dinv[c], 0.0);
#pragma unroll
      for (int r = c + 1; r < M; ++r) {
        double2 s = make_double2(0.0, 0.0);
#pragma unroll
        for (int k = c; k < r; ++k) s = cfma(L[r + k * M], Li[k + c * M], s);
        Li[r + c * M] = make_double2(-s.x * dinv[r], -s.y * dinv[r]);
      }
    }
#pragma unroll
    for (int c = 0; c < M; ++c) {
#pragma unroll
      for (int r = c; r < M; ++r) {
        double2 s = make_double2(0.0, 0.0);
#pragma unroll
        for (int k = r; k < M; ++k) s = cfmac(Li[k + r * M], Li[k + c * M], s);
        O[r + c * M] = s;
        O[c + r * M] = cconj(s);
      }
      O[c + c * M].y = 0.0;
    }
    return true;
  }
}

struct NaiveArgs {
  int64_t nb;
  int64_t J;
  int iters;
  double alpha, beta, eps;
  const double2* X;    // [bin][t][m]
  const double2* a;    // [bin][M]
  const double2* b;    // [bin][M]
  const double2* Rp;   // [bin][M*M]
  double* r_h;         // [bin][t] in/out
  double* r_u;         // [bin][t] in/out
  double* lambda;      // [bin] in/out
  double2* scratch;    // [bin][t] (T_a, T_b)
  double* traj_r_h;
  double* traj_r_u;
  double* traj_lambda;
  unsigned long long* err;
};

// One CTA per frequency bin runs every iteration (solver_naive.hpp:427-435
// with the per-bin fusion of :319-386); threads stride over the bin's frames.
// EMU (NT = 64): the CTA holds the frames a 128-thread CTA would, thread tid those of
// threads tid and tid + 64, keeps their two lambda accumulators apart (rounds of even
// and odd parity) and leaves four warp partials in the 128-thread layout's order, so
// every bit equals the 128-thread result: the CTA size may then follow the batch
// size (J = 320 runs 5 exact rounds of 64 instead of 3 of 128 with half of the last
// idle) without a sharded run differing from an unsharded one.
// (for M <= 4 the kernel is held to 168 registers -- 8 bytes of spills at M = 4 -- so
// twelve warps, three per SM sub-partition, share an SM: six 64-thread or three
// 128-thread CTAs)
template <int M, int NT, bool EMU = false>
__global__ void __launch_bounds__(NT, M <= 4 ? 384 / NT : 1) k_naive(NaiveArgs P) {
  static_assert(!EMU || NT == 64, "EMU emulates 128 threads with 64");
  constexpr int NW = EMU ? 4 : NT / 32;  // warp partials of the (emulated) layout
  __shared__ double2 sa[M], sb[M], sw[M], su[M];
  __shared__ double2 sRp[M * M], sRut[M * M];
  __shared__ double sc[2];  // beta0 = Re b^H R~_u b, beta1 = Re b^H R~_u^{-1} b
  __shared__ double red[2][NW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t bin = blockIdx.x;
  const int64_t J = P.J;
  for (int k = tid; k < M * M; k += NT) sRp[k] = P.Rp[bin * M * M + k];
  if (tid < M) {
    sa[tid] = P.a[bin * M + tid];
    sb[tid] = P.b[bin * M + tid];
  }
  double lam = P.lambda[bin];
  const double inv_a2 = 1.0 / (P.alpha + 2.0);
  __syncthreads();
  for (int it = 0; it < P.iters; ++it) {
    // Per-bin constants of the E-step with the previous lambda.
    for (int k = tid; k < M * M; k += NT) {
      const int r = k % M, c = k / M;
      sRut[k] = cadd(sRp[k], cmul(cscale(sb[r], lam), cconj(sb[c])));  // R' + lambda b b^H
    }
    __syncthreads();
    if (tid == 0) {
      double2 Ru[M * M], Rui[M * M];
#pragma unroll
      for (int k = 0; k < M * M; ++k) Ru[k] = sRut[k];
      if (!herm_pd_inverse<M>(Ru, Rui)) {
        report_error(P.err, bin * J, kErrMStepSingular);
#pragma unroll
        for (int k = 0; k < M * M; ++k) Rui[k] = make_double2(0.0, 0.0);
      }
      double2 s0 = make_double2(0.0, 0.0), s1 = s0;
#pragma unroll
      for (int r = 0; r < M; ++r) {
        double2 w = make_double2(0.0, 0.0), u = w;
#pragma unroll
        for (int j = 0; j < M; ++j) {
          w = cfma(Ru[r + j * M], sb[j], w);
          u = cfma(Rui[r + j * M], sb[j], u);
        }
        sw[r] = w;
        su[r] = u;
        s0 = cfmac(sb[r], w, s0);
        s1 = cfmac(sb[r], u, s1);
      }
      sc[0] = s0.x;
      sc[1] = s1.x;
    }
    __syncthreads();
    const double beta0 = sc[0], beta1 = sc[1];
    double acc = 0.0;
    [[maybe_unused]] double acc_hi = 0.0;  // EMU: the accumulator of emulated thread tid + 64
    [[maybe_unused]] int round = 0;
    for (int64_t t = tid; t < J; t += NT, ++round) {
      const int64_t slot = bin * J + t;
      const double rh = P.r_h[slot], ru = P.r_u[slot];
      double2 x[M];
#pragma unroll
      for (int m = 0; m < M; ++m) x[m] = P.X[slot * M + m];
      // R_x = r~_h a a^H + r~_u R~_u (solver_naive.hpp:201-206)
      double2 Rx[M * M], Ri[M * M];
#pragma unroll
      for (int c = 0; c < M; ++c) {
        const double2 ac = cscale(cconj(sa[c]), rh);
#pragma unroll
        for (int r = c; r < M; ++r) {
          const double2 ut = sRut[r + c * M];
          Rx[r + c * M] = cadd(cmul(sa[r], ac), make_double2(ru * ut.x, ru * ut.y));
        }
#pragma unroll
        for (int r = 0; r < c; ++r) Rx[r + c * M] = cconj(Rx[c + r * M]);
      }
      if (!herm_pd_inverse<M>(Rx, Ri)) {  // solver_naive.hpp:207-209
        report_error(P.err, slot, kErrEStepSingular);
#pragma unroll
        for (int k = 0; k < M * M; ++k) Ri[k] = make_double2(0.0, 0.0);
      }
      // za = R_x^{-1} a, z = R_x^{-1} x, zw = R_x^{-1} w, zb = R_x^{-1} b
      double2 za[M], z[M], zw[M], zb[M];
#pragma unroll
      for (int r = 0; r < M; ++r) {
        double2 s1 = make_double2(0.0, 0.0), s2 = s1, s3 = s1, s4 = s1;
#pragma unroll
        for (int c = 0; c < M; ++c) {
          const double2 ri = Ri[r + c * M];
          s1 = cfma(ri, sa[c], s1);
          s2 = cfma(ri, x[c], s2);
          s3 = cfma(ri, sw[c], s3);
          s4 = cfma(ri, sb[c], s4);
        }
        za[r] = s1;
        z[r] = s2;
        zw[r] = s3;
        zb[r] = s4;
      }
      double ara = 0.0, wzw = 0.0, bzb = 0.0;
      double2 xra = make_double2(0.0, 0.0), wz = xra, bz = xra;
#pragma unroll
      for (int r = 0; r < M; ++r) {
        ara += cmulc(sa[r], za[r]).x;
        xra = cfmac(x[r], za[r], xra);
        wzw += cmulc(sw[r], zw[r]).x;
        wz = cfmac(sw[r], z[r], wz);
        bzb += cmulc(sb[r], zb[r]).x;
        bz = cfmac(sb[r], z[r], bz);
      }
      // r^_h (solver_naive.hpp:211-220)
      const double hrh = rh - rh * rh * ara + cnorm(make_double2(rh * xra.x, rh * xra.y));
      const double ru2 = ru * ru;
      const double q = ru * beta0 - ru2 * wzw + ru2 * cnorm(wz);
      // tr(R_x^{-1} R~_u) and z^H R~_u z
      double tr = 0.0, zuz = 0.0;
#pragma unroll
      for (int r = 0; r < M; ++r) {
        double2 uz = make_double2(0.0, 0.0);
#pragma unroll
        for (int c = 0; c < M; ++c) {
          tr += cmul(Ri[r + c * M], sRut[c + r * M]).x;
          uz = cfma(sRut[r + c * M], z[c], uz);
        }
        zuz += cmulc(z[r], uz).x;
      }
      const double Ta = ru * M - ru2 * tr + ru2 * zuz;
      const double Tb = ru * beta1 - ru2 * bzb + ru2 * cnorm(bz);
      P.r_h[slot] = std_max((hrh + P.beta) * inv_a2, P.eps);  // solver_naive.hpp:333-334
      P.scratch[slot] = make_double2(Ta, Tb);
      if (EMU && (round & 1)) acc_hi += q / ru; else acc += q / ru;
    }
    acc = warp_sum(acc);
    const int buf = it & 1;
    if constexpr (EMU) {
      acc_hi = warp_sum(acc_hi);
      if (lane == 0) {
        red[buf][warp] = acc;
        red[buf][warp + 2] = acc_hi;
      }
    } else {
      if (lane == 0) red[buf][warp] = acc;
    }
    __syncthreads();
    double total = 0.0;
    for (int w = 0; w < NW; ++w) total += red[buf][w];
    const double lam_new = std_max(total / static_cast<double>(J), P.eps);
    const double d = lam_new - lam;
    const double den = fma(d, beta1, 1.0);
    // R_u = R~_u + d b b^H (solver_naive.hpp:357-368) is PD iff R~_u is and
    // 1 + d b^H R~_u^-1 b > 0 (a NaN lambda fails too, as the reference's
    // !(x > 0) tests do): the reference's "m_step: singular R^(u)" at this M-step
    // (keyed at the bin's last frame: the reference finishes the bin's E-step,
    // whose singular-frame errors take precedence, before its M-step)
    if (tid == 0 && !(den > 0.0)) report_error(P.err, bin * J + (J - 1), kErrMStepSingular);
    const double f = d / den;
    lam = lam_new;
    for (int64_t t = tid; t < J; t += NT) {
      const int64_t slot = bin * J + t;
      const double2 ab = P.scratch[slot];
      P.r_u[slot] = std_max(fma(-f, ab.y, ab.x) / M, P.eps);
      if (P.traj_r_h) {
        const int64_t o = static_cast<int64_t>(it) * P.nb * J + slot;
        P.traj_r_h[o] = P.r_h[slot];
        P.traj_r_u[o] = P.r_u[slot];
      }
    }
    if (P.traj_lambda && tid == 0) P.traj_lambda[static_cast<int64_t>(it) * P.nb + bin] = lam;
    __syncthreads();
  }
  if (tid == 0) P.lambda[bin] = lam;
}

}  // namespace rcscm
