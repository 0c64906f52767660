// accel.cuh -- K2: the on-chip Algorithm 2 iteration kernel (sm_100a).
//
// Reference: solver_accel.hpp:183-240 (detail::run_accelerated with
// second_stage = true), i.e. per iteration
//   gamma = r~_h / (r~_u + r~_h rho~_aa) (+ gamma_fault)            :67-76, :213
//   r_h   = max((gamma (r~_u + gamma |rho~_ax|^2) + beta)/(alpha+2), eps)  :134-141
//   lambda= max((1/J) sum_t [gamma |s_ab|^2 + |s_bx - gamma conj(s_ab) rho~_ax|^2 / r~_u], eps) :143-158
//   rho   = tau + sigma-terms / lambda_new                             :113-129
//   r_u   = max((gamma rho_aa q + rho_xx - 2 gamma Re(rho~_ax conj rho_ax))/M, eps) :160-176
//
// Mapping: one CTA (CL == 1) or one thread-block cluster of CL CTAs per
// frequency bin. Each thread owns SPT slots of the bin and keeps every
// per-slot quantity (r_h, r_u, rho~_ax, tau_ax, s_ab*s_bx, s_bx, tau_xx, |s_bx|^2)
// in REGISTERS for all iterations: HBM is touched once to load (56 B/slot) and
// once to store (16 B/slot). The only cross-slot dependency -- lambda's sum over
// frames -- is a fixed-order tree: in-thread pairwise sum, a warp total on the
// FP64 tensor core (DMMA), a zero-padded 8-way block tree (+ DSMEM exchange
// across the cluster), so results are deterministic and independent of how
// many GPUs the bins are sharded over.
//
// Latency structure: the lambda reduction is the only serial step of an
// iteration, so each iteration computes the lambda-critical values first,
// starts the warp reduction, and overlaps it with everything that does not
// depend on the new lambda -- r_h and the two coefficients of r_u, which is
// affine in 1/lambda_new (M r_u = P0 + P1/lambda_new). After the block total only
// three FMAs per slot remain (r_u, and rho_ax for the next iteration).
//
// Instruction budget per slot-iteration (47 canonical flops): 35 FP64 ops
// (DFMA/DMUL) + 1 MUFU.RCP64H; floors run on the integer ALUs. The reference's
// two divisions share one reciprocal (inv = 1/(D r~_u) gives gamma = r~_h r~_u inv
// and 1/r~_u = D inv); gamma_fault rides in an FMA; 1/M is folded into the
// per-slot constants (exact for power-of-two M); `max(v, eps)` keeps the
// reference's std::max semantics.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace rcscm {

struct AccelArgs {
  int64_t nb;
  int64_t J;
  int iters;
  double inv_M;
  double k1;  // 1 / (alpha + 2)
  double k2;  // beta / (alpha + 2)
  double eps;
  double gamma_fault;
  const double2* sigma_ab;  // [bin]
  const double* tau_aa;     // [bin]
  const double2* sigma_bx;  // [bin][t]
  const double2* tau_ax;    // [bin][t]
  const double* tau_xx;     // [bin][t]
  double* r_h;              // [bin][t] in/out
  double* r_u;              // [bin][t] in/out
  double* lambda;           // [bin]    in/out
  double* traj_r_h;         // optional [it][bin][t]
  double* traj_r_u;
  double* traj_lambda;      // optional [it][bin]
};

// std::max(v, eps) of the reference (returns v unless v < eps) for eps > 0,
// evaluated as a signed 64-bit compare of the bit patterns: IEEE doubles of
// either sign order like their two's-complement images against a positive eps
// (negative v and -0.0 map below eps, +NaN stays NaN as in std::max). Keeps the
// floor on the integer ALUs instead of the FP64 pipe.
__device__ __forceinline__ double floor_eps(double v, double eps) {
  const long long iv = __double_as_longlong(v), ie = __double_as_longlong(eps);
  return __longlong_as_double(iv < ie ? ie : iv);
}

// Sum of the 32 lanes' values, returned in every lane, on the FP64 tensor
// core: DMMA m8n8k4 with B = 1 leaves in lane l the sum of its 4-lane group
// g_{l/4}; one shuffle round transposes the 8 group sums into the k index and
// two more DMMAs (B = 1) add them. ~90 cycles of latency on B200 against
// ~180 for a 5-step shuffle butterfly (measured: DMMA 26, SHFL.f64+DADD 36).
// Multiplications by 1 are exact and the DMMA's internal order is fixed, so
// the result is deterministic and identical in every lane.
__device__ __forceinline__ double dmma_ones(double a) {
  double d0;
  [[maybe_unused]] double d1;
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
      : "=d"(d0), "=d"(d1)
      : "d"(a), "d"(1.0), "d"(0.0), "d"(0.0));
  return d0;
}
__device__ __forceinline__ double warp_total_mma(double v, int lane) {
  const double g = dmma_ones(v);  // lane l: sum of lanes 4*(l/4) .. +3
  const int src = (lane & 3) << 2;
  const double lo = __shfl_sync(0xffffffffu, g, src);       // g_{l%4}
  const double hi = __shfl_sync(0xffffffffu, g, src + 16);  // g_{l%4 + 4}
  return dmma_ones(lo) + dmma_ones(hi);
}

// Sum of the (zero-padded) first 4 per-warp partials (CTAs of <= 128 threads).
__device__ __forceinline__ double block_total4(const double* red) {
  const double2* r = reinterpret_cast<const double2*>(red);
  const double2 a = r[0], b = r[1];
  return (a.x + a.y) + (b.x + b.y);
}

// Sum of the (zero-padded) 8 per-warp partials: four broadcast LDS.128 and a
// fixed 3-level tree, identical in every thread.
__device__ __forceinline__ double block_total8(const double* red) {
  const double2* r = reinterpret_cast<const double2*>(red);
  const double2 a = r[0], b = r[1], c = r[2], d = r[3];
  return ((a.x + a.y) + (b.x + b.y)) + ((c.x + c.y) + (d.x + d.y));
}

// FULL: every thread's SPT slots are inside the bin chunk (NT * SPT == chunk),
// so no per-slot masks. TRAJ: record r_h / r_u / lambda after every iteration.
// SMEMC: the four per-slot constants used only after the lambda reduction
// (tau_ax, s_ab*s_bx, tau_xx/M, |s_bx|^2/M: 48 B/slot) live in dynamic shared
// memory ([k][tid] planes, conflict-free) instead of registers, which roughly
// halves the register footprint and doubles the resident warps per SM.
// LB3: launch bounds of 128 threads x 3 CTAs/SM (<= 170 registers) instead of
// one 256-thread CTA's worth, trading a little ILP for resident warps.
// DIRECT: form r_u after the reduction from rho with the new lambda (8 FP64 ops
// per slot, the reference's own order) instead of the affine P0 + P1/lambda
// split (10 ops, but all but 3 of them overlap the reduction).
template <int SPT, int CL, bool FULL, bool TRAJ, bool SMEMC, bool LB3 = false, bool DIRECT = false>
__global__ void __launch_bounds__(LB3 ? 128 : 256, LB3 ? 3 : (SMEMC ? 2 : 1)) k_accel(AccelArgs P) {
  namespace cg = cooperative_groups;
  constexpr int kMaxWarps = 256 / 32;
  __shared__ __align__(16) double red[2][kMaxWarps];  // zero-padded warp partials
  // cluster exchange: cl_vals[buf][r] receives rank r's CTA partial, cl_bar[buf]
  // counts the CL arrivals (double-buffered by iteration parity)
  __shared__ __align__(16) double cl_vals[2][16];
  __shared__ __align__(8) unsigned long long cl_bar[2];
  extern __shared__ double2 dyn[];
  const int NT = blockDim.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t bin = blockIdx.x / CL;
  const int rank = (CL > 1) ? static_cast<int>(blockIdx.x % CL) : 0;
  const int64_t J = P.J;
  const int64_t Jc = (J + CL - 1) / CL;
  const int64_t t0 = rank * Jc;
  const int64_t t_end = min(J, t0 + Jc);
  const int64_t base = bin * J;
  const double inv_M = P.inv_M;
  // shared planes (SMEMC): tax[k][tid], cc[k][tid] (double2), txx[k][tid], dd[k][tid] (double)
  double2* s_tax = dyn;
  double2* s_cc = dyn + SPT * NT;
  double* s_txx = reinterpret_cast<double*>(dyn + 2 * SPT * NT);
  double* s_dd = s_txx + SPT * NT;

  const double2 sab = P.sigma_ab[bin];
  const double s2 = cnorm(sab);  // |sigma_ab|^2
  const double taa = P.tau_aa[bin];
  double lam = P.lambda[bin];
  double il = 1.0 / lam;
  double raa = fma(s2, il, taa);  // rho_aa (solver_accel.hpp:122)

  // per-slot state: rh, ru evolve; rax = rho~_ax carried; the rest is constant.
  // txx and dd are pre-scaled by 1/M (exact for M = 2, 4, 8, 16).
  constexpr int SR = SMEMC ? 1 : SPT;  // register copies of the constants
  double rh[SPT], ru[SPT], txx[SR], dd[SR];
  double2 rax[SPT], tax[SR], cc[SR], sbx[SPT];
  bool valid[SPT];
#pragma unroll
  for (int k = 0; k < SPT; ++k) {
    const int64_t t = t0 + static_cast<int64_t>(k) * NT + tid;
    valid[k] = FULL || t < t_end;
    const int64_t s = base + (valid[k] ? t : t0);
    rh[k] = P.r_h[s];
    ru[k] = P.r_u[s];
    sbx[k] = P.sigma_bx[s];
    const double2 tk = P.tau_ax[s];
    const double xk = P.tau_xx[s] * inv_M;
    const double2 ck = cmul(sab, sbx[k]);   // sigma_ab * sigma_bx
    const double dk = cnorm(sbx[k]) * inv_M;  // |sigma_bx|^2 / M
    rax[k] = make_double2(fma(ck.x, il, tk.x), fma(ck.y, il, tk.y));
    if constexpr (SMEMC) {
      s_tax[k * NT + tid] = tk;
      s_cc[k * NT + tid] = ck;
      s_txx[k * NT + tid] = xk;
      s_dd[k * NT + tid] = dk;
    } else {
      tax[k] = tk;
      cc[k] = ck;
      txx[k] = xk;
      dd[k] = dk;
    }
  }

  if (tid < 2 * kMaxWarps) (&red[0][0])[tid] = 0.0;
  if constexpr (CL > 1) {
    if (tid < 2) {
      const unsigned lb = static_cast<unsigned>(__cvta_generic_to_shared(&cl_bar[tid]));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(lb), "r"(CL) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    cg::this_cluster().sync();  // every peer's barriers exist before the first remote arrive
  } else {
    __syncthreads();
  }
  const double invJ = 1.0 / static_cast<double>(J);
  const double m2M = -2.0 * inv_M;
  const double taaM = taa * inv_M, s2M = s2 * inv_M;
  const double fault = P.gamma_fault;
  for (int it = 0; it < P.iters; ++it) {
    const int buf = it & 1;
    // (1) lambda-critical values first: gamma, 1/r~_u and the residual norm
    //     (solver_accel.hpp:67-76, :143-158).
    double g[SPT], term[SPT];
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      const double D = fma(rh[k], raa, ru[k]);  // r~_u + r~_h rho~_aa
      const double inv = rcp_pos(D * ru[k]);
      const double gk = fma(rh[k] * inv, ru[k], fault);  // gamma (+ gamma_fault)
      const double iru = D * inv;                         // 1 / r~_u
      // resid = s_bx - gamma conj(s_ab) rho~_ax
      const double2 e = cmulc(sab, rax[k]);
      const double rx = fma(-gk, e.x, sbx[k].x);
      const double ry = fma(-gk, e.y, sbx[k].y);
      const double rr = fma(rx, rx, ry * ry);
      // per-slot lambda term, independent across slots (no serial accumulator)
      term[k] = (FULL || valid[k]) ? fma(gk, s2, rr * iru) : 0.0;
      g[k] = gk;
    }
    // fixed pairwise tree over the thread's slots, then the warp butterfly
#pragma unroll
    for (int w = 1; w < SPT; w <<= 1) {
#pragma unroll
      for (int k = 0; k + w < SPT; k += 2 * w) term[k] += term[k + w];
    }
    const double part = warp_total_mma(term[0], lane);
    if (lane == 0) red[buf][warp] = part;
    // (2) everything that does not need the new lambda, overlapping the
    //     reduction: r_h (solver_accel.hpp:134-141) and the two halves of the
    //     r_u update, which is affine in 1/lambda_new (:160-176 with :121-127):
    //       M r_u = P0 + P1 / lambda_new,
    //       P0 = g q tau_aa + tau_xx - 2 g Re(rho~_ax conj tau_ax)
    //       P1 = g q |s_ab|^2 + |s_bx|^2 - 2 g Re(rho~_ax conj(s_ab s_bx))
    //     (stored pre-scaled by 1/M; q = r~_u + g |rho~_ax|^2).
    double p0[SPT], p1[SPT];
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      if constexpr (DIRECT) {
        const double q = fma(g[k], cnorm(rax[k]), ru[k]);
        const double gq = g[k] * q;
        rh[k] = floor_eps(fma(gq, P.k1, P.k2), P.eps);
        p0[k] = gq;             // gamma q
        p1[k] = g[k] * m2M;     // -2 gamma / M
        continue;
      }
      double2 tk, ck;
      double xk, dk;
      if constexpr (SMEMC) {
        tk = s_tax[k * NT + tid];
        ck = s_cc[k * NT + tid];
        xk = s_txx[k * NT + tid];
        dk = s_dd[k * NT + tid];
      } else {
        tk = tax[k];
        ck = cc[k];
        xk = txx[k];
        dk = dd[k];
      }
      const double q = fma(g[k], cnorm(rax[k]), ru[k]);
      const double gq = g[k] * q;
      rh[k] = floor_eps(fma(gq, P.k1, P.k2), P.eps);
      const double m2g = g[k] * m2M;                              // -2 gamma / M
      const double re0 = fma(rax[k].x, tk.x, rax[k].y * tk.y);    // Re(rho~_ax conj tau_ax)
      const double re1 = fma(rax[k].x, ck.x, rax[k].y * ck.y);    // Re(rho~_ax conj(s_ab s_bx))
      p0[k] = fma(m2g, re0, fma(gq, taaM, xk));
      p1[k] = fma(m2g, re1, fma(gq, s2M, dk));
    }
    __syncthreads();
    double total = 0.0;
    if constexpr (CL == 1) {
      total = NT <= 128 ? block_total4(red[buf]) : block_total8(red[buf]);
    } else {
      // CTA partial -> cluster: lanes r < CL of warp 0 store this CTA's partial
      // into cl_vals[buf][rank] of CTA r (st.shared::cluster) and arrive on its
      // cl_bar[buf] with release semantics; every thread then waits on the local
      // barrier (acquire) and sums the CL partials in rank order -- the same
      // fixed tree in every CTA. One DSMEM write latency instead of a
      // cluster-wide barrier plus a remote read.
      const double c = block_total8(red[buf]);
      if (warp == 0 && lane < CL) {
        const unsigned lv = static_cast<unsigned>(__cvta_generic_to_shared(&cl_vals[buf][rank]));
        const unsigned lb = static_cast<unsigned>(__cvta_generic_to_shared(&cl_bar[buf]));
        unsigned rv, rb;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rv) : "r"(lv), "r"(lane));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(lb), "r"(lane));
        asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(rv), "d"(c) : "memory");
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rb) : "memory");
      }
      {
        const unsigned lb = static_cast<unsigned>(__cvta_generic_to_shared(&cl_bar[buf]));
        const unsigned parity = static_cast<unsigned>((it >> 1) & 1);
        unsigned done = 0;
        while (!done) {
          asm volatile(
              "{\n .reg .pred p;\n"
              " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
              " selp.u32 %0, 1, 0, p;\n}"
              : "=r"(done)
              : "r"(lb), "r"(parity)
              : "memory");
        }
      }
      double v[CL];
#pragma unroll
      for (int r = 0; r < CL; ++r) v[r] = cl_vals[buf][r];
#pragma unroll
      for (int w = 1; w < CL; w <<= 1) {
#pragma unroll
        for (int r = 0; r + w < CL; r += 2 * w) v[r] += v[r + w];
      }
      total = v[0];
    }
    // (3) the short tail that needs lambda_new
    lam = floor_eps(total * invJ, P.eps);
    il = rcp_pos(lam);
    raa = fma(s2, il, taa);
    const double raaM = raa * inv_M;
#pragma unroll
    for (int k = 0; k < SPT; ++k) {
      double2 tk, ck;
      double xk = 0.0, dk = 0.0;
      if constexpr (SMEMC) {
        tk = s_tax[k * NT + tid];
        ck = s_cc[k * NT + tid];
        if constexpr (DIRECT) {
          xk = s_txx[k * NT + tid];
          dk = s_dd[k * NT + tid];
        }
      } else {
        tk = tax[k];
        ck = cc[k];
        if constexpr (DIRECT) {
          xk = txx[k];
          dk = dd[k];
        }
      }
      const double2 nax = make_double2(fma(ck.x, il, tk.x), fma(ck.y, il, tk.y));  // rho_ax, lambda_new
      if constexpr (DIRECT) {
        // solver_accel.hpp:167-173 with rho_xx / M = tau_xx/M + |s_bx|^2/M / lambda
        const double rxx = fma(dk, il, xk);
        const double re = fma(rax[k].x, nax.x, rax[k].y * nax.y);  // Re(rho~_ax conj(rho_ax))
        ru[k] = floor_eps(fma(p1[k], re, fma(p0[k], raaM, rxx)), P.eps);
      } else {
        ru[k] = floor_eps(fma(p1[k], il, p0[k]), P.eps);
      }
      rax[k] = nax;
    }
    if constexpr (TRAJ) {
#pragma unroll
      for (int k = 0; k < SPT; ++k) {
        if (valid[k]) {
          const int64_t t = t0 + static_cast<int64_t>(k) * NT + tid;
          const int64_t o = static_cast<int64_t>(it) * P.nb * J + base + t;
          P.traj_r_h[o] = rh[k];
          P.traj_r_u[o] = ru[k];
        }
      }
      if (rank == 0 && tid == 0) P.traj_lambda[static_cast<int64_t>(it) * P.nb + bin] = lam;
    }
  }
#pragma unroll
  for (int k = 0; k < SPT; ++k) {
    if (valid[k]) {
      const int64_t t = t0 + static_cast<int64_t>(k) * NT + tid;
      P.r_h[base + t] = rh[k];
      P.r_u[base + t] = ru[k];
    }
  }
  if (rank == 0 && tid == 0) P.lambda[bin] = lam;
  if constexpr (CL > 1) {
    // No CTA leaves while a peer may still be writing into its shared memory.
    cooperative_groups::this_cluster().sync();
  }
}

}  // namespace rcscm
