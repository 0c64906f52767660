// accel_stream.cuh -- K2s: Algorithm 2 for bins too long for the on-chip kernel
// (J > 16 CTAs x 256 threads x 8 slots = 32768 frames), streaming the per-slot
// state through HBM every iteration (sm_100a).
//
// Reference: solver_accel.hpp:183-240, the loop the reference runs for ANY
// number of frames (update_lambda :143-158 is a plain loop over t). One
// iteration is two launches over a (bins x frame-chunks) grid:
//   k_stream_term    gamma, the scaled residual and lambda's per-slot term from
//                    the current iterate (r_h, r_u in HBM, rho~ from tau / sigma
//                    and the current lambda), reduced per chunk in a fixed tree
//                    -> partial[bin][chunk];
//   k_stream_update  every CTA sums its bin's chunk partials in a fixed order
//                    (identical bits in every CTA of the bin), forms
//                    lambda_new, recomputes its slots' gamma / q from the
//                    unchanged iterate and writes r_h and r_u (the on-chip
//                    kernel's DIRECT arithmetic, slot for slot); lambda goes to
//                    the other buffer of a ping-pong pair, so no CTA reads a
//                    lambda another CTA of the same launch has already updated.
// Deterministic (no atomics, fixed trees) and independent of how bins are
// sharded; per iteration it moves 56 B/slot in and 56 + 16 B/slot out of HBM
// (the on-chip kernel: 0.7 B per slot-iteration), the price of bins that do not
// fit a cluster's registers and shared memory.
#pragma once

#include "accel.cuh"

namespace rcscm {

struct StreamAccelArgs {
  int64_t nb, J, chunks;  // chunks of kStreamChunk frames per bin
  int iters;
  double inv_M, k1, k2, eps, gamma_fault;
  const double2* sigma_ab;  // [bin]
  const double* tau_aa;     // [bin]
  const double2* sigma_bx;  // [bin][t]
  const double2* tau_ax;    // [bin][t]
  const double* tau_xx;     // [bin][t]
  const double* r_h_in;     // [bin][t] current iterate (may alias r_h)
  const double* r_u_in;
  double* r_h;              // [bin][t] out
  double* r_u;
  const double* lam_old;    // [bin] lambda of the current iterate
  const double* il_old;     // [bin] its reciprocal as K2 carries it (null: 1 / lam_old, the first iteration)
  double* lam_new;          // [bin]
  double* il_new;           // [bin]
  double* partial;          // [bin][chunk]
  double* traj_r_h;         // optional [it][bin][t] (written by the update of iteration `it`)
  double* traj_r_u;
  double* traj_lambda;      // optional [it][bin]
  int it;
};

constexpr int kStreamNT = 256, kStreamSPT = 4, kStreamChunk = kStreamNT * kStreamSPT;

// Per-bin scalars of K2's prologue (accel.cuh), from the resident precompute.
struct StreamBin {
  double s2, taa, lam, il, raa;
  double2 sabT;  // s_ab / |s_ab|^2 (1 when s_ab = 0: the literal residual)
  bool scaled;
};
__device__ __forceinline__ StreamBin stream_bin(const StreamAccelArgs& P, int64_t bin) {
  StreamBin b;
  const double2 sab = P.sigma_ab[bin];
  b.taa = P.tau_aa[bin];
  b.s2 = cnorm(sab);
  b.scaled = b.s2 > 0.0;
  const double cs = b.scaled ? 1.0 / b.s2 : 0.0;
  b.sabT = b.scaled ? make_double2(sab.x * cs, sab.y * cs) : make_double2(1.0, 0.0);
  b.lam = P.lam_old[bin];
  if (P.il_old) {  // K2's loop form: the carried reciprocal, rho_aa = tau_aa + s2 / lambda
    b.il = P.il_old[bin];
    b.raa = b.taa + b.il * b.s2;
  } else {  // K2's prologue form
    b.il = 1.0 / b.lam;
    b.raa = fma(b.s2, b.il, b.taa);
  }
  return b;
}

// gamma, 1/r~_u and lambda's term of one slot (K2 phase 1, accel.cuh)
__device__ __forceinline__ void stream_phase1(const StreamBin& b, double gamma_fault, double rh, double ru,
                                              double2 ck, double2 rax, double& g, double& term) {
  const double D = fma(rh, b.raa, ru);
  const double inv = rcp_pos(D * ru);
  g = fma(rh * inv, ru, gamma_fault);
  const double iru = D * inv;
  const double rx = b.scaled ? fma(-g, rax.x, ck.x) : ck.x;
  const double ry = b.scaled ? fma(-g, rax.y, ck.y) : ck.y;
  const double rr = fma(rx, rx, ry * ry);
  term = b.scaled ? fma(rr, iru, g) : rr * iru;
}

__global__ void __launch_bounds__(kStreamNT) k_stream_term(StreamAccelArgs P) {
  __shared__ __align__(16) double red[8];
  const int64_t bin = blockIdx.x, chunk = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t J = P.J, base = bin * J;
  const StreamBin b = stream_bin(P, bin);
  const double ilc = b.il * b.s2;
  double term[kStreamSPT];
#pragma unroll
  for (int k = 0; k < kStreamSPT; ++k) {
    const int64_t t = chunk * kStreamChunk + static_cast<int64_t>(k) * kStreamNT + tid;
    term[k] = 0.0;
    if (t < J) {
      const int64_t s = base + t;
      const double2 ck = cmul(b.sabT, P.sigma_bx[s]), tk = P.tau_ax[s];
      const double2 rax = make_double2(fma(ck.x, ilc, tk.x), fma(ck.y, ilc, tk.y));
      double g;
      stream_phase1(b, P.gamma_fault, P.r_h_in[s], P.r_u_in[s], ck, rax, g, term[k]);
    }
  }
  // fixed trees: in-thread pairwise, warp total, block over the 8 warps
  const double v = (term[0] + term[1]) + (term[2] + term[3]);
  const double w = warp_total(v);
  if (lane == 0) red[warp] = w;
  __syncthreads();
  if (tid == 0) P.partial[bin * P.chunks + chunk] = block_total8(red);
}

__global__ void __launch_bounds__(kStreamNT) k_stream_update(StreamAccelArgs P) {
  const int64_t bin = blockIdx.x, chunk = blockIdx.y;
  const int tid = threadIdx.x;
  const int64_t J = P.J, base = bin * J;
  const StreamBin b = stream_bin(P, bin);
  // lambda_new from the bin's chunk partials -- warp 0: lane l sums chunks l,
  // l + 32, ... in order, then the fixed warp butterfly (the same bits in every
  // CTA of the bin) -- then K2's floor and speculative reciprocal
  __shared__ double s_total;
  if (tid < 32) {
    double acc = 0.0;
    for (int64_t c = tid; c < P.chunks; c += 32) acc += P.partial[bin * P.chunks + c];
    acc = warp_sum(acc);
    if (tid == 0) s_total = acc;
  }
  __syncthreads();
  const double total = s_total;
  const double invJ = 1.0 / static_cast<double>(J);
  const double lraw = total * (b.scaled ? b.s2 * invJ : invJ);
  const bool fl = below_eps(lraw, P.eps);
  const double lam = fl ? P.eps : lraw;
  const double il = fl ? rcp_pos(P.eps) : rcp_pos(lraw);
  const double ilc_old = b.il * b.s2, ilc = il * b.s2;
  const double raaM = fma(ilc, P.inv_M, b.taa * P.inv_M);
  const double m2M = -2.0 * P.inv_M;
  if (chunk == 0 && tid == 0) {
    P.lam_new[bin] = lam;
    P.il_new[bin] = il;
    if (P.traj_lambda) P.traj_lambda[static_cast<int64_t>(P.it) * P.nb + bin] = lam;
  }
#pragma unroll
  for (int k = 0; k < kStreamSPT; ++k) {
    const int64_t t = chunk * kStreamChunk + static_cast<int64_t>(k) * kStreamNT + tid;
    if (t >= J) continue;
    const int64_t s = base + t;
    const double2 sb = P.sigma_bx[s], tk = P.tau_ax[s];
    const double2 ck = cmul(b.sabT, sb);
    const double2 rax = make_double2(fma(ck.x, ilc_old, tk.x), fma(ck.y, ilc_old, tk.y));
    const double rh = P.r_h_in[s], ru = P.r_u_in[s];
    double g, term;
    stream_phase1(b, P.gamma_fault, rh, ru, ck, rax, g, term);
    // K2 phase 2 / 3 (DIRECT): r_h, then r_u with rho at lambda_new
    const double q = fma(g, cnorm(rax), ru);
    const double gq = g * q;
    const double rh_new = floor_eps(fma(gq, P.k1, P.k2), P.eps);
    const double p1 = g * m2M;
    const double2 nax = make_double2(fma(ck.x, ilc, tk.x), fma(ck.y, ilc, tk.y));
    const double xk = P.tau_xx[s] * P.inv_M, dk = cnorm(sb) * P.inv_M;
    const double rxx = fma(dk, il, xk);
    const double re = fma(rax.x, nax.x, rax.y * nax.y);
    const double ru_new = floor_eps(fma(p1, re, fma(gq, raaM, rxx)), P.eps);
    P.r_h[s] = rh_new;
    P.r_u[s] = ru_new;
    if (P.traj_r_h) {
      const int64_t o = static_cast<int64_t>(P.it) * P.nb * J + s;
      P.traj_r_h[o] = rh_new;
      P.traj_r_u[o] = ru_new;
    }
  }
}

}  // namespace rcscm
