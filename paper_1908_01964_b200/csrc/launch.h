// launch.h -- host-side launchers of the rcscm kernels, one translation unit
// per kernel family (setup_launch.cu, accel_launch.cu, naive_launch.cu,
// stream_launch.cu). Each returns cudaSuccess or the launch error; M-templated
// kernels are dispatched at run time over the supported channel counts.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "accel.cuh"
#include "accel1.cuh"
#include "naive.cuh"
#include "setup.cuh"
#include "stream.cuh"

namespace rcscm {

// true if this build has kernels for M channels (1..8 and 16)
bool mics_supported(int M);

// K1a + K1b (build_noise_scm): mean powers, then per-bin R', b, R'^+, a, lambda0.
cudaError_t launch_setup(cudaStream_t s, const DevProblem& P, double rank_tol, double eps);
// K1b in MODE 1: lambda0 only from a given R' (init_params).
cudaError_t launch_lambda0(cudaStream_t s, const DevProblem& P, double eps);
// K1: slot stream kernel (INIT: r_h0 / r_u0, PRE: sigma / tau).
cudaError_t launch_slots(cudaStream_t s, const DevProblem& P, bool init, bool pre, double eps);

// K2 launch configuration (cluster size, threads, slots per thread).
// CTAs per SM the launch bounds of the tuned single-CTA K2 target (128-thread
// bounds x 4: <= 128 registers, 8 CTAs of 64 threads per SM). With the scalar
// carried state (k_accel SST) a slot needs 12 registers; measured on B200, C3:
// 4.60 ms at 3 (168 registers) against 4.38 ms at 4, 128 utterances.
#ifndef RCSCM_K2_MINB1
#define RCSCM_K2_MINB1 4
#endif

struct AccelCfg {
  int cl, nt, spt;
  bool full;  // nt * spt == chunk: no per-slot masks
  int smem;   // per-slot constants in shared memory (k_accel SMEMC: 0 none, 1 all, 2 tax/txx/dd)
  int minb;   // 128-thread x minb-CTA launch bounds (k_accel MINB), CL == 1 and nt <= 128 only
  bool direct;  // r_u from rho(lambda_new) after the reduction (k_accel DIRECT), MINB path only
  bool f32;     // complex64 / FP32 per-slot arithmetic
  int prem = 0;  // fused precompute for M = prem mics (k_accel PREM; 0 = read K1's arrays)
  int we = 0;    // one-warp CTAs emulating a CTA of `we` warps (k_accel WE; fused shapes only)
};
// Chooses the configuration for J frames; env RCSCM_ACCEL_SPT / RCSCM_ACCEL_CL /
// RCSCM_ACCEL_SMEM / RCSCM_ACCEL_MINB force a choice (tuning). Returns cl == 0 when J exceeds the on-chip capacity.
AccelCfg choose_accel_cfg(int64_t J, bool f32 = false);
cudaError_t launch_accel(cudaStream_t s, const AccelArgs& A, const AccelCfg& cfg);
// true if K2 can fuse the sigma / tau precompute for this configuration (the
// tuned single-CTA complex128 variant, M in {2, 4, 8}); env RCSCM_FUSE_PRE=0
// disables it
bool accel_fusable(const AccelCfg& cfg, int M);
// For a fused configuration over nb bins: switch to one-warp CTAs (k_accel WE)
// where that layout is instantiated and the batch fills the GPU with them;
// every result stays bitwise the same (env RCSCM_ACCEL_W1 = the fewest bins
// that take it, 0 disables it)
void accel_one_warp(AccelCfg& cfg, int64_t nb);
// Algorithm 2 streaming the iterate through HBM for bins longer than the on-chip
// kernel holds (accel_stream.cuh; needs K1's sigma / tau arrays, complex128):
// 2 launches per iteration; partial: [nb][accel_stream_chunks(J)], lam_buf: 4 nb.
int64_t accel_stream_chunks(int64_t J);
cudaError_t launch_accel_stream(cudaStream_t s, const AccelArgs& A, double* partial, double* lam_buf, int* n_launch);

cudaError_t launch_naive(cudaStream_t s, int M, const NaiveArgs& N);
// K6: Algorithm 1 (first-stage acceleration), every iteration in one launch
cudaError_t launch_accel1(cudaStream_t s, int M, const Accel1Args& A);

cudaError_t launch_wiener(cudaStream_t s, int M, const WienerArgs& W, bool from_x, bool noise);
// K1b MODE 2: log pseudo-determinant of each bin's R' (P.logpdet)
cudaError_t launch_logpdet(cudaStream_t s, const DevProblem& P);
// O(1)-per-slot objective partial sums (np = grid size written to *np)
cudaError_t launch_objective_fast(cudaStream_t s, ObjFastArgs O, int64_t* np);
// objective partial sums (np = grid size written to *np) and the final sum
cudaError_t launch_objective(cudaStream_t s, int M, ObjArgs O, int64_t* np);
cudaError_t launch_sum_partials(cudaStream_t s, const double* partial, int64_t n, double* out);
cudaError_t launch_sum_rows(cudaStream_t s, const double* partial, int rows, int64_t n, double* out);
// reference I x J column-major (leading dimension ld, 0 = I) <-> device [bin][t]
// (B blocks of I bins)
cudaError_t launch_to_bt(cudaStream_t s, const double* src, double* dst, int64_t B, int64_t I, int64_t J,
                         int64_t ld = 0);
cudaError_t launch_to_ij(cudaStream_t s, const double* src, double* dst, int64_t B, int64_t I, int64_t J,
                         int64_t ld = 0);
cudaError_t launch_to_ij_c(cudaStream_t s, const double2* src, double2* dst, int64_t B, int64_t I, int64_t J);
// double2 layout change: to_bt: src (i, t) at i + t*ld -> dst[i*J + t]; else the inverse
cudaError_t launch_transpose_c(cudaStream_t s, const double2* src, double2* dst, int64_t I, int64_t J, int64_t ld,
                               bool to_bt);
cudaError_t launch_fp64_probe(cudaStream_t s, int blocks, int iters, double* out);

// ILRMA (ilrma.cu): sphering, NMF / IP sweeps, scale normalisation, inverses
struct IlrmaArgs {
  int64_t I, J;
  int K;
  const double2* X;  // [bin][t][m] (whitened)
  double2* W;        // [bin][M*M]
  double2* A;        // [bin][M*M]
  double* T;         // [n][I x K col-major]
  double* V;         // [n][K x J col-major]
  double* P;         // [n][bin][t]
  double* Pt;        // [n][t][bin] (the same powers, transposed for the V update)
  double* partial;   // [n][ilrma_partials(I, J)]
  double* mu;        // [n]
  double2* ucov;     // [bin][n][M*M] IP weighted covariances
  unsigned long long* err;
};
int64_t ilrma_partials(int64_t I, int64_t J);
cudaError_t launch_sphere(cudaStream_t s, int M, const double2* X, int64_t I, int64_t J, double2* Q, double2* Xw);
cudaError_t launch_ilrma_powers(cudaStream_t s, const IlrmaArgs& A, int M);
cudaError_t launch_ilrma_nmf(cudaStream_t s, const IlrmaArgs& A, int M);     // K <= 16
cudaError_t launch_ilrma_ip_scale(cudaStream_t s, const IlrmaArgs& A, int M);  // IP sweep + powers + scaling
cudaError_t launch_ilrma_inverse(cudaStream_t s, const IlrmaArgs& A, int M);
// W = W_ilrma Q, Am = W^{-1} per bin (A.W holds W_ilrma)
cudaError_t launch_ilrma_fold(cudaStream_t s, const IlrmaArgs& A, int M, const double2* Q, double2* W, double2* Am);
// power[n][i] = ||(W_i X_i)_n||^2 ||Am_i(:, n)||^2
cudaError_t launch_target_power(cudaStream_t s, int M, const double2* X, const double2* W, const double2* Am,
                                int64_t I, int64_t J, double* power);

// STFT (stft.cu): cached batched cuFFT plans (D2Z and Z2D of length n, batch rows)
struct StftPlan {
  int fwd = 0, inv = 0;  // cufftHandle
  int n = 0;
  int64_t batch = 0;
  StftPlan() = default;
  StftPlan(const StftPlan&) = delete;
  StftPlan& operator=(const StftPlan&) = delete;
  ~StftPlan();
  void reset();
  cudaError_t ensure(int win, int64_t batch, cudaStream_t s);
};
// x: (ch, p) at ch + p*M (planar: ch*len + p); window[win]; scratch
// frames[J*M*win], spec[J*M*(win/2+1)]; X out: [bin][frame][mic] (stft.hpp:50-88)
cudaError_t launch_stft_analyze(cudaStream_t s, StftPlan& plan, const double* x, int64_t len, int M, int win,
                                int hop, int64_t J, const double* window, double* frames, double2* spec,
                                double2* X, bool planar = false);
// X: [bin][frame][mic], B bins; dual_n = WOLA dual window / win; out (ch, p) at
// ch + p*M (planar: ch*len + p) (stft.hpp:92-129)
cudaError_t launch_stft_synthesize(cudaStream_t s, StftPlan& plan, const double2* X, int64_t B, int64_t J, int M,
                                   int win, int hop, int64_t len, const double* dual_n, double2* spec,
                                   double* frames, double* out, bool planar = false);
cudaError_t launch_fp32_probe(cudaStream_t s, int blocks, int iters, double* out);

// complex64 (FP32) mode
cudaError_t launch_slots_pre_f32(cudaStream_t s, const DevProblem& P, const float2* Xf, float2* sbx, float2* tax,
                                 float* txx);
cudaError_t launch_wiener_f32(cudaStream_t s, int M, const WienerArgsF32& W, bool from_x);
cudaError_t launch_d2f(cudaStream_t s, const double* src, float* dst, int64_t n);
cudaError_t launch_f2d(cudaStream_t s, const float* src, double* dst, int64_t n);

}  // namespace rcscm
