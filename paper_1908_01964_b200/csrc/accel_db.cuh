// accel_db.cuh -- K2d: Algorithm 2 on-chip with TWO bins in flight per cluster
// (sm_100a). Reference: solver_accel.hpp:183-240, the same per-slot arithmetic
// as k_accel's scalar carried state (accel.cuh, SST2).
//
// Why: a bin that needs a cluster pays, every iteration, a serial chain -- warp
// total, CTA total, DSMEM exchange, 1 / lambda -- during which its CTAs have
// nothing to issue, and the CTAs of a cluster wait for the slowest of them
// (each shares its SM with a CTA of another cluster at a random phase). Here a
// cluster of CL CTAs owns the bin pair (2p, 2p + 1): every thread holds 4 slots
// of each, and the two bins run half an iteration apart in program order,
//   wait lambda_A -> phase 3 (A) -> phase 1 (A) -> send A's partial
//   wait lambda_B -> phase 3 (B) -> phase 1 (B) -> send B's partial
// so A's reduction, exchange and peer skew overlap B's arithmetic and vice
// versa. No CTA-wide barrier in the loop: each warp leaves its partial in shared
// memory and counts itself in with an acq_rel atomic; the warp that arrives last
// sums the (zero-padded) partials in block_total8's fixed order and sends the CTA
// partial to every peer (st.async + mbarrier complete_tx, as k_accel). Every
// sum is a fixed tree, so results are deterministic and a bin's result does not
// depend on its partner or on how bins are sharded (the two roles run the same
// inlined arithmetic; tested bitwise).
#pragma once

#include <cooperative_groups.h>

#include "accel.cuh"

namespace rcscm {

constexpr int kDbSlots = 4;  // slots per thread and bin

struct DbBin {
  double rh[kDbSlots], ru[kDbSlots], n2[kDbSlots], b2[kDbSlots], xk[kDbSlots], ak[kDbSlots];
  double g[kDbSlots], q[kDbSlots];  // gamma and q = r~_u + gamma |rho~|^2, kept across the wait
  double lam, il, ilc, raa;         // lambda, 1 / lambda, |s_ab|^2 / lambda, rho_aa
  double s2, taa, taaM, lscale;     // |s_ab|^2, tau_aa, tau_aa / M, the bin total's scale
  bool scaled;
};

__device__ __forceinline__ unsigned db_count_in(unsigned* cnt) {
  unsigned old;
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(cnt));
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(a) : "memory");
  return old;
}

template <int CL, bool FULL, int PREM>
__global__ void __launch_bounds__(256, 2) k_accel_db(AccelArgs P) {
  namespace cg = cooperative_groups;
  constexpr int S = kDbSlots;
  __shared__ __align__(16) double red[2][2][8];      // [bin][buf][warp], zero-padded
  __shared__ unsigned cnt[2];                         // warps counted in, per bin
  __shared__ __align__(16) double cl_vals[2][2][16];  // [bin][buf][rank]
  __shared__ __align__(8) unsigned long long cl_bar[2][2];
  __shared__ double2 pR[2][PREM * PREM], pb[2][PREM], pp[2][PREM];
  const int NT = blockDim.x, nwarps = NT >> 5;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t pair = blockIdx.x / CL;
  const int rank = static_cast<int>(blockIdx.x % CL);
  const int64_t bins[2] = {2 * pair, min(2 * pair + 1, P.nb - 1)};
  const bool store[2] = {true, 2 * pair + 1 < P.nb};  // an odd last bin runs twice, stored once
  const int64_t J = P.J;
  const int64_t Jc = (J + CL - 1) / CL;
  const int64_t t0 = rank * Jc;
  const int64_t t_end = min(J, t0 + Jc);
  const int64_t ldp = P.ld_p;
  const double inv_M = P.inv_M;
  const double invJ = 1.0 / static_cast<double>(J);
  const double k1 = P.k1, k2 = P.k2, eps = P.eps, fault = P.gamma_fault;
  const double m2M = -2.0 * inv_M;
  const double il_eps = rcp_pos(P.eps);

  bool valid[S];
  int64_t tt[S];
#pragma unroll
  for (int k = 0; k < S; ++k) {
    const int64_t t = t0 + static_cast<int64_t>(k) * NT + tid;
    valid[k] = FULL || t < t_end;
    tt[k] = valid[k] ? t : t0;
  }

  // per-bin prologue of K1 (k_pre): R'^+, b and R'^+ a in shared memory
#pragma unroll
  for (int w = 0; w < 2; ++w) {
    const int64_t bin = bins[w];
    for (int k = tid; k < PREM * PREM; k += NT) pR[w][k] = P.Rpp_in[bin * PREM * PREM + k];
    if (tid < PREM) {
      pb[w][tid] = P.b_in[bin * PREM + tid];
      double2 s = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < PREM; ++k)
        s = cfma(P.Rpp_in[bin * PREM * PREM + tid + k * PREM], __ldg(P.a_in + bin * PREM + k), s);
      pp[w][tid] = s;
    }
  }
  if (tid < 2 * 2 * 8) (&red[0][0][0])[tid] = 0.0;
  if (tid < 2) cnt[tid] = 0u;
  if (tid < 4) {
    const unsigned lb = static_cast<unsigned>(__cvta_generic_to_shared(&cl_bar[tid >> 1][tid & 1]));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(lb) : "memory");
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();

  DbBin B[2];
#pragma unroll
  for (int w = 0; w < 2; ++w) {
    DbBin& X = B[w];
    const int64_t bin = bins[w];
    const int64_t base = bin * J;
    double2 ab = make_double2(0.0, 0.0), aa = make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < PREM; ++k) {
      const double2 ak = __ldg(P.a_in + bin * PREM + k);
      ab = cfmac(ak, pb[w][k], ab);
      aa = cfmac(ak, pp[w][k], aa);
    }
    const double2 sab = ab;
    X.taa = std_max(aa.x, 0.0);
    if (rank == 0 && tid == 0 && P.sigma_ab_w && store[w]) {
      P.sigma_ab_w[bin] = sab;
      P.tau_aa_w[bin] = X.taa;
    }
    X.s2 = cnorm(sab);
    X.lam = P.lambda_in[bin];
    X.il = 1.0 / X.lam;
    X.scaled = X.s2 > 0.0;
    const double cs = X.scaled ? 1.0 / X.s2 : 0.0;
    const double2 sabT = X.scaled ? make_double2(sab.x * cs, sab.y * cs) : make_double2(1.0, 0.0);
    X.ilc = __dmul_rn(X.il, X.s2);
    X.raa = fma(X.s2, X.il, X.taa);
    X.taaM = X.taa * inv_M;
    X.lscale = X.scaled ? X.s2 * invJ : invJ;
#pragma unroll
    for (int k = 0; k < S; ++k) {
      const int64_t s = base + tt[k];
      const int64_t sp = ldp ? bin + tt[k] * ldp : s;
      X.rh[k] = __ldg(P.r_h_in + sp);
      X.ru[k] = __ldg(P.r_u_in + sp);
      double2 xv[PREM];
#pragma unroll
      for (int m = 0; m < PREM; ++m) xv[m] = __ldg(P.X + s * PREM + m);
      double2 sb, tk;
      double txx;
      slot_forms<PREM>(xv, pb[w], pp[w], pR[w], sb, tk, txx);
      if (P.sigma_bx_w && valid[k] && store[w]) {
        P.sigma_bx_w[s] = sb;
        P.tau_ax_w[s] = tk;
        P.tau_xx_w[s] = txx;
      }
      // the scalar carried state of k_accel (SST): c = s_ab s_bx / |s_ab|^2,
      // rho~ = tau_ax + c |s_ab|^2 / lambda, (|rho~|^2, b2 = -2 Re(conj(c) rho~))
      const double2 ck = cmul(sabT, sb);
      double2 r0;
      r0.x = fma(ck.x, X.ilc, tk.x);
      r0.y = fma(ck.y, X.ilc, tk.y);
      X.n2[k] = cnorm(r0);
      X.b2[k] = -2.0 * fma(ck.x, r0.x, ck.y * r0.y);
      X.ak[k] = cnorm(ck);
      X.xk[k] = txx * inv_M;
    }
  }
  cg::this_cluster().sync();  // every peer's barriers exist before the first remote arrive

  // phase (1): gamma, 1 / r~_u, q and the lambda term's numerator; the thread's
  // sum by two FMA chains; the warp total; then count in, and the last warp of
  // the CTA sends the CTA partial to every peer
  auto phase1_send = [&](DbBin& X, int w, int buf) {
    double u[S], ir[S];
#pragma unroll
    for (int k = 0; k < S; ++k) {
      const double D = fma(X.rh[k], X.raa, X.ru[k]);
      const double inv = rcp_pos(D * X.ru[k]);
      const double gk = fma(X.rh[k] * inv, X.ru[k], fault);
      ir[k] = D * inv;
      const double q = fma(gk, X.n2[k], X.ru[k]);
      const double un = fma(gk, q + X.b2[k], X.ak[k]);  // |s_bx|^2 alone when s_ab = 0
      u[k] = (FULL || valid[k]) ? (X.scaled ? un : X.ak[k]) : 0.0;
      X.g[k] = gk;
      X.q[k] = q;
    }
    double ce = u[0] * ir[0], co = u[1] * ir[1];
    ce = fma(u[2], ir[2], ce);
    co = fma(u[3], ir[3], co);
    const double part = warp_total(ce + co);
    unsigned old = 0;
    if (lane == 0) {
      red[w][buf][warp] = part;
      old = db_count_in(&cnt[w]);
    }
    old = __shfl_sync(0xffffffffu, old, 0);
    if ((old + 1) % nwarps == 0) {  // this warp is the last of the round: every partial is visible
      __syncwarp();
      const double c = block_total8(red[w][buf]);
      const unsigned lb = static_cast<unsigned>(__cvta_generic_to_shared(&cl_bar[w][buf]));
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(lb), "r"(CL * 8) : "memory");
      if (lane < CL) {
        const unsigned lv = static_cast<unsigned>(__cvta_generic_to_shared(&cl_vals[w][buf][rank]));
        unsigned rv, rb;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rv) : "r"(lv), "r"(lane));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(lb), "r"(lane));
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(rv), "d"(c),
                     "r"(rb)
                     : "memory");
      }
    }
  };

  // wait for the bin's CL partials of iteration it, lambda and its per-bin
  // scalars (solver_accel.hpp:143-158), then phase (3): r_h, r_u and the state
  auto wait_phase3 = [&](DbBin& X, int w, int it) {
    const int buf = it & 1;
    const unsigned lb = static_cast<unsigned>(__cvta_generic_to_shared(&cl_bar[w][buf]));
    const unsigned parity = static_cast<unsigned>((it >> 1) & 1);
    unsigned done = 0;
    while (!done) {
      asm volatile(
          "{\n .reg .pred p;\n"
          " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
          " selp.u32 %0, 1, 0, p;\n}"
          : "=r"(done)
          : "r"(lb), "r"(parity)
          : "memory");
    }
    double v[CL];
#pragma unroll
    for (int r = 0; r < CL; ++r) v[r] = cl_vals[w][buf][r];
#pragma unroll
    for (int s = 1; s < CL; s <<= 1) {
#pragma unroll
      for (int r = 0; r + s < CL; r += 2 * s) v[r] += v[r + s];
    }
    const double lraw = __dmul_rn(v[0], X.lscale);
    const double ilr = rcp_pos(lraw);
    const bool fl = below_eps(lraw, eps);
    X.lam = fl ? eps : lraw;
    X.il = fl ? il_eps : ilr;
    const double ilc = __dmul_rn(X.il, X.s2);
    X.raa = __dadd_rn(X.taa, ilc);
    const double ds = __dsub_rn(ilc, X.ilc);  // change of |s_ab|^2 / lambda (0 when s_ab = 0)
    X.ilc = ilc;
    const double raaM = fma(ilc, inv_M, X.taaM);
    const double xA = __dmul_rn(X.scaled ? ilc : X.il, inv_M);
    const double hds = -0.5 * ds, m2ds = -2.0 * ds;
#pragma unroll
    for (int k = 0; k < S; ++k) {
      const double gq = X.g[k] * X.q[k];
      X.rh[k] = floor_eps(fma(gq, k1, k2), eps);
      const double p1 = X.g[k] * m2M;
      const double rxx = fma(X.ak[k], xA, X.xk[k]);
      const double re = fma(hds, X.b2[k], X.n2[k]);  // Re(rho~ conj(rho~ + c ds))
      X.ru[k] = floor_eps(fma(p1, re, fma(gq, raaM, rxx)), eps);
      X.b2[k] = fma(m2ds, X.ak[k], X.b2[k]);
      X.n2[k] = fma(hds, X.b2[k], re);
    }
  };

  const int iters = P.iters;
  if (iters > 0) {
    phase1_send(B[0], 0, 0);
    phase1_send(B[1], 1, 0);
  }
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    const bool more = it + 1 < iters;
    wait_phase3(B[0], 0, it);
    if (more) phase1_send(B[0], 0, (it + 1) & 1);
    wait_phase3(B[1], 1, it);
    if (more) phase1_send(B[1], 1, (it + 1) & 1);
  }

#pragma unroll
  for (int w = 0; w < 2; ++w) {
    if (!store[w]) continue;
    const int64_t bin = bins[w];
#pragma unroll
    for (int k = 0; k < S; ++k) {
      if (valid[k]) {
        const int64_t sp = ldp ? bin + tt[k] * ldp : bin * J + tt[k];
        P.r_h[sp] = B[w].rh[k];
        P.r_u[sp] = B[w].ru[k];
      }
    }
    if (rank == 0 && tid == 0) P.lambda[bin] = B[w].lam;
  }
  // No CTA leaves while a peer may still be writing into its shared memory.
  cg::this_cluster().sync();
}

}  // namespace rcscm
