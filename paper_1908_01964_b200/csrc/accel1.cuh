// accel1.cuh -- K6: Algorithm 1 (first-stage acceleration) on the GPU, sm_100a.
//
// Reference: solver_accel.hpp:80-109 (rho_first_stage), :183-240
// (detail::run_accelerated with second_stage = false), :245-250
// (run_algorithm1). Per iteration and bin:
//   gamma = r~_h / (r~_u + r~_h rho~_aa) (+ gamma_fault)              :67-76, :213
//   r_h   = max((gamma (r~_u + gamma |rho~_ax|^2) + beta)/(alpha+2), eps)  :134-141
//   lambda= max((1/J) sum_t [gamma |s_ab|^2 + |s_bx - gamma conj(s_ab) rho~_ax|^2 / r~_u], eps) :143-158
//   R_u   = R' + lambda b b^H, R_u^{-1} by Cholesky (Eigen::LLT semantics)  :93-99
//   rho_aa = Re a^H R_u^{-1} a, rho_ax = (R_u^{-1} a)^H x, rho_xx = Re x^H R_u^{-1} x :100-107
//   r_u   = max((gamma rho_aa q + rho_xx - 2 gamma Re(rho~_ax conj rho_ax))/M, eps) :160-176
// with s_ab = a^H b and s_bx = b^H x (precompute_sigma, :33-43). Unlike
// Algorithm 2 it needs R' (not R'^+) and an M x M inverse per bin per iteration:
// O(I M^3 + I J M^2) per iteration. It is the third backend of the reference's
// verify suite (tools/rcscm.cpp:223-275, acceptance.cpp:34-65), not a
// throughput path: one CTA per bin runs every iteration, threads stride over
// the bin's frames (any J), x is re-read from global memory (L2) each
// iteration, and the per-slot carried quantities (rho~_ax, gamma, s_bx) live in
// device scratch. The lambda sum is a fixed-order per-thread + warp butterfly +
// warp-partial tree, so results are deterministic.
#pragma once

#include "common.cuh"

namespace rcscm {

struct Accel1Args {
  int64_t nb, J;
  int iters;
  double alpha2, beta;  // alpha + 2, beta
  double eps, gamma_fault;
  const double2* X;   // [bin][t][m]
  const double2* a;   // [bin][M]
  const double2* b;   // [bin][M]
  const double2* Rp;  // [bin][M*M]
  double* r_h;        // [bin][t] in/out
  double* r_u;        // [bin][t] in/out
  double* lambda;     // [bin]    in/out
  double2* rho_ax;    // [bin][t] scratch: rho_ax of the current parameters
  double2* sigma_bx;  // [bin][t] scratch
  double* gamma;      // [bin][t] scratch
  double* traj_r_h;   // optional [it][bin][t]
  double* traj_r_u;
  double* traj_lambda;  // optional [it][bin]
  unsigned long long* err;
};

// R^{-1} of a Hermitian PD M x M matrix in shared memory by one thread:
// Cholesky R = L L^H on the lower triangle (Eigen::LLT: fail when a pivot is
// not > 0), then R^{-1} = L^{-H} L^{-1}. L and O are shared scratch (M*M).
template <int M>
__device__ bool llt_inverse_1t(const double2* R, double2* L, double2* O) {
  for (int k = 0; k < M * M; ++k) L[k] = make_double2(0.0, 0.0);
  for (int k = 0; k < M; ++k) {
    double x = R[k + k * M].x;
    for (int j = 0; j < k; ++j) x -= cnorm(L[k + j * M]);
    if (!(x > 0.0)) return false;
    const double lkk = sqrt(x);
    L[k + k * M] = make_double2(lkk, 0.0);
    const double dk = 1.0 / lkk;
    for (int i = k + 1; i < M; ++i) {
      double2 s = R[i + k * M];
      for (int j = 0; j < k; ++j) s = csub(s, cmul(L[i + j * M], cconj(L[k + j * M])));
      L[i + k * M] = cscale(s, dk);
    }
  }
  // L^{-1} (lower triangular) column by column into O by forward substitution
  for (int c = 0; c < M; ++c) {
    for (int r = 0; r < M; ++r) O[r + c * M] = make_double2(0.0, 0.0);
    O[c + c * M] = make_double2(1.0 / L[c + c * M].x, 0.0);
    for (int r = c + 1; r < M; ++r) {
      double2 s = make_double2(0.0, 0.0);
      for (int k = c; k < r; ++k) s = cfma(L[r + k * M], O[k + c * M], s);
      const double d = 1.0 / L[r + r * M].x;
      O[r + c * M] = make_double2(-s.x * d, -s.y * d);
    }
  }
  // R^{-1} = L^{-H} L^{-1}: copy L^{-1} into L's storage, form the product in O
  for (int k = 0; k < M * M; ++k) L[k] = O[k];
  for (int c = 0; c < M; ++c) {
    for (int r = c; r < M; ++r) {
      double2 s = make_double2(0.0, 0.0);
      for (int k = r; k < M; ++k) s = cfmac(L[k + r * M], L[k + c * M], s);
      O[r + c * M] = s;
      O[c + r * M] = cconj(s);
    }
    O[c + c * M].y = 0.0;
  }
  return true;
}

template <int M, int NT>
__global__ void __launch_bounds__(NT) k_accel1(Accel1Args P) {
  __shared__ double2 sa[M], sb[M], sRp[M * M], sRu[M * M], sL[M * M], sRi[M * M], sri_a[M];
  __shared__ double s_rho_aa;
  __shared__ double red[2][NT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t bin = blockIdx.x;
  const int64_t J = P.J;
  for (int k = tid; k < M * M; k += NT) sRp[k] = P.Rp[bin * M * M + k];
  if (tid < M) {
    sa[tid] = P.a[bin * M + tid];
    sb[tid] = P.b[bin * M + tid];
  }
  __syncthreads();
  // sigma_ab = a^H b (solver_accel.hpp:39)
  double2 sab = make_double2(0.0, 0.0);
  for (int k = 0; k < M; ++k) sab = cfmac(sa[k], sb[k], sab);
  const double s2 = cnorm(sab);
  const double2 csab = cconj(sab);
  double lam = P.lambda[bin];

  // rho_first_stage for lambda: R_u, its inverse, R_u^{-1} a, rho_aa (one thread)
  auto first_stage = [&](double l) {
    if (tid == 0) {
      int ok = 1;
      if (!(l > 0.0)) {  // solver_accel.hpp:90-92
        report_error(P.err, bin * J, kErrFirstStageLambda);
        ok = 0;
      } else {
        for (int k = 0; k < M * M; ++k) {
          const int r = k % M, c = k / M;
          sRu[k] = cadd(sRp[k], cmul(cscale(sb[r], l), cconj(sb[c])));  // R' + lambda b b^H
        }
        if (!llt_inverse_1t<M>(sRu, sL, sRi)) {  // solver_accel.hpp:95-97
          report_error(P.err, bin * J, kErrFirstStageSingular);
          ok = 0;
        }
      }
      if (!ok)
        for (int k = 0; k < M * M; ++k) sRi[k] = make_double2(0.0, 0.0);
      double2 ara = make_double2(0.0, 0.0);
      for (int r = 0; r < M; ++r) {
        double2 s = make_double2(0.0, 0.0);
        for (int c = 0; c < M; ++c) s = cfma(sRi[r + c * M], sa[c], s);
        sri_a[r] = s;
        ara = cfmac(sa[r], s, ara);
      }
      s_rho_aa = ara.x;
    }
    __syncthreads();
  };

  // line 4: sigma_bx and rho_ax for the initial parameters (no rho_xx)
  first_stage(lam);
  double rho_aa = s_rho_aa;
  for (int64_t t = tid; t < J; t += NT) {
    const int64_t slot = bin * J + t;
    double2 sbx = make_double2(0.0, 0.0), rax = sbx;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const double2 xm = P.X[slot * M + m];
      sbx = cfmac(sb[m], xm, sbx);
      rax = cfmac(sri_a[m], xm, rax);
    }
    P.sigma_bx[slot] = sbx;
    P.rho_ax[slot] = rax;
  }
  __syncthreads();

  for (int it = 0; it < P.iters; ++it) {
    const double trho_aa = rho_aa;
    // gamma, r_h and the lambda terms (solver_accel.hpp:67-76, :134-158)
    double acc = 0.0;
    for (int64_t t = tid; t < J; t += NT) {
      const int64_t slot = bin * J + t;
      const double rh = P.r_h[slot], ru = P.r_u[slot];
      const double2 trax = P.rho_ax[slot];
      const double g = rh / (ru + rh * trho_aa) + P.gamma_fault;
      P.gamma[slot] = g;
      P.r_h[slot] = std_max((g * (ru + g * cnorm(trax)) + P.beta) / P.alpha2, P.eps);
      const double2 sbx = P.sigma_bx[slot];
      const double2 gc = cscale(csab, g);
      const double2 resid = csub(sbx, cmul(gc, trax));
      acc += g * s2 + cnorm(resid) / ru;
    }
    acc = warp_sum(acc);
    const int buf = it & 1;
    if (lane == 0) red[buf][warp] = acc;
    __syncthreads();
    double total = 0.0;
    for (int w = 0; w < NT / 32; ++w) total += red[buf][w];
    lam = std_max(total / static_cast<double>(J), P.eps);
    // rho with the new lambda (line 14) and r_u (solver_accel.hpp:160-176)
    first_stage(lam);
    rho_aa = s_rho_aa;
    for (int64_t t = tid; t < J; t += NT) {
      const int64_t slot = bin * J + t;
      double2 x[M];
#pragma unroll
      for (int m = 0; m < M; ++m) x[m] = P.X[slot * M + m];
      double2 rax = make_double2(0.0, 0.0), xx = rax;
#pragma unroll
      for (int r = 0; r < M; ++r) {
        rax = cfmac(sri_a[r], x[r], rax);
        double2 acc2 = make_double2(0.0, 0.0);
#pragma unroll
        for (int c = 0; c < M; ++c) acc2 = cfma(sRi[r + c * M], x[c], acc2);
        xx = cfmac(x[r], acc2, xx);
      }
      const double g = P.gamma[slot];
      const double ru = P.r_u[slot];
      const double2 trax = P.rho_ax[slot];
      const double val = (g * rho_aa * (ru + g * cnorm(trax)) + xx.x - 2.0 * g * cmulc(rax, trax).x) / M;
      P.r_u[slot] = std_max(val, P.eps);
      P.rho_ax[slot] = rax;
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
