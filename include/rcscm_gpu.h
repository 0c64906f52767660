/*
 * rcscm_gpu.h -- C ABI of the B200 (sm_100a) rank-constrained SCM hot path.
 *
 * Drop-in boundary for the reference's C++ entry points (all paths relative to
 * /root/reference/proj/include/rcscm/):
 *
 *   rcscm_gpu_build_noise_scm   replaces  build_noise_scm       model.hpp:58-90
 *   rcscm_gpu_init_params       replaces  init_params           model.hpp:95-124
 *   rcscm_gpu_map_objective     replaces  map_objective         model.hpp:129-157
 *   rcscm_gpu_run_naive         replaces  run_naive             solver_naive.hpp:412-450
 *   rcscm_gpu_run_algorithm1    replaces  run_algorithm1        solver_accel.hpp:245-250
 *   rcscm_gpu_run_algorithm2    replaces  run_algorithm2        solver_accel.hpp:254-258
 *   rcscm_gpu_run_accel         stage 1 / 2 -> run_algorithm1 / 2 (one accelerated symbol)
 *   rcscm_gpu_build_inputs      build_noise_scm + init_params     model.hpp:58-124
 *   rcscm_gpu_extract_target    replaces  extract_target        wiener.hpp:19-43
 *   rcscm_gpu_extract_noise     replaces  extract_noise         wiener.hpp:46-53
 *   rcscm_gpu_stft_analyze      replaces  stft_analyze          stft.hpp:50-88
 *   rcscm_gpu_stft_synthesize   replaces  stft_synthesize       stft.hpp:92-129
 *   rcscm_gpu_sphere            replaces  sphere                ilrma.hpp:53-73
 *   rcscm_gpu_run_ilrma         replaces  run_ilrma             ilrma.hpp:145-240
 *   rcscm_gpu_extract           replaces  cmd_extract's pipeline tools/rcscm.cpp:158-221
 *
 * Plain pointers and sizes only; no CUDA or Eigen types cross the boundary.
 * Host buffers use the reference's Eigen column-major complex128 layouts:
 *   X, image, noise  : [i][t][m]  complex interleaved   (Spectrogram::bins[i], M x J col-major)
 *   a, b             : [i][m]     complex
 *   R', R'^+, W, A   : [i][r + c*M] complex             (M x M col-major per bin)
 *   r_h, r_u         : element (i, t) at i + t*I        (Eigen MatR, I x J)
 *   dry              : element (i, t) at i + t*I, complex
 *   lambda           : [i]
 *   T (NmfModel::T[n_h], I x K) : i + k*I ;  V (NmfModel::V[n_h], K x J) : k + t*K
 *   waveform samples : (ch, p) at ch + p*M             (Waveform::samples, M x len col-major)
 *
 * Error contract (types.hpp:20-30, tools/rcscm.cpp:22-25): functions return
 *   RCSCM_OK (0), RCSCM_INVALID_INPUT (2, InvalidInputError),
 *   RCSCM_NUMERICAL (3, NumericalError, message names "bin i, frame t"),
 *   RCSCM_CUDA_ERROR (4), RCSCM_UNSUPPORTED (5);
 * the message of the last failure on the calling thread is rcscm_gpu_last_error().
 *
 * Threading: calls are synchronous (outputs are in the caller's buffers on
 * return). One context per host thread; a context is not thread-safe.
 */
#ifndef RCSCM_GPU_H
#define RCSCM_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RCSCM_OK 0
#define RCSCM_INVALID_INPUT 2
#define RCSCM_NUMERICAL 3
#define RCSCM_CUDA_ERROR 4
#define RCSCM_UNSUPPORTED 5

#define RCSCM_C128 0
#define RCSCM_C64 1

typedef struct rcscm_gpu_ctx rcscm_gpu_ctx;

typedef struct {
  int device;    /* CUDA device ordinal */
  int precision; /* RCSCM_C128 (reference-exact) or RCSCM_C64 (FP32 mode) */
  void* stream;  /* cudaStream_t to launch on; NULL = context-owned stream */
  /* Optional device list: with num_devices > 1 the solver entry
   * points (run_naive / run_algorithm1 / run_algorithm2 without objective or
   * trajectory) and extract_target / extract_noise shard contiguous, balanced
   * bin ranges over devices[0..num_devices) -- one host thread and stream per
   * device, inputs sliced straight from the caller's buffers, each range's
   * results copied back into its own (strided, for I x J col-major arrays)
   * slice of the caller's outputs. No collective: bins are independent, and
   * results are bitwise equal to the single-device call. devices[0] replaces
   * `device`; `stream` applies to devices[0] only. NULL / 0 / 1: one device. */
  const int* devices;
  int num_devices;
} rcscm_gpu_config;

/* model.hpp:16-25 RcscmInputs (host pointers, reference layout). */
typedef struct {
  int64_t num_bins;
  int64_t frames;
  int mics;
  int n_h;
  const double* a;
  const double* R_prime;
  const double* R_prime_pinv;
  const double* b;
} rcscm_inputs;

/* model.hpp:29-33 RcscmParams (host pointers, reference layout). */
typedef struct {
  double* r_h;
  double* r_u;
  double* lambda;
} rcscm_params;

/* model.hpp:36-39 Hyperparams */
typedef struct {
  double alpha;
  double beta;
} rcscm_hyper;

/* solver_naive.hpp:14-22 SolverOptions. `threads` is accepted for source
 * compatibility; the CUDA grid replaces parallel_for (results do not depend on it). */
typedef struct {
  int iters;
  int compute_objective;
  int record_trajectory;
  double rel_obj_tol;
  int threads;
  double eps_var;
  double gamma_fault;
} rcscm_solver_opts;

/* solver_naive.hpp:24-29 SolverResult extras (every pointer optional / NULL):
 *   objective    [iters + 1]            (needs compute_objective)
 *   iter_seconds [iters]                (CUDA-event time of each iteration's kernel(s))
 *   traj_r_h, traj_r_u [iters][I*J]     (reference layout per snapshot)
 *   traj_lambda  [iters][I]
 * n_objective / n_iters receive the number of entries written. */
typedef struct {
  double* objective;
  int* n_objective;
  double* iter_seconds;
  int* n_iters;
  double* traj_r_h;
  double* traj_r_u;
  double* traj_lambda;
} rcscm_result;

/* ---- context ------------------------------------------------------------ */
int rcscm_gpu_create(const rcscm_gpu_config* cfg, rcscm_gpu_ctx** out);
void rcscm_gpu_destroy(rcscm_gpu_ctx* ctx);
const char* rcscm_gpu_last_error(void);
/* Number of CUDA kernels this context has launched so far. */
int64_t rcscm_gpu_launch_count(const rcscm_gpu_ctx* ctx);

/* ---- reference entry points (host buffers) ------------------------------ */
/* model.hpp:58-90 */
int rcscm_gpu_build_noise_scm(rcscm_gpu_ctx* ctx, int64_t I, int64_t J, int M,
                              const double* X, const double* W, const double* A,
                              int n_h, double rank_tol, double* a, double* R_prime,
                              double* R_prime_pinv, double* b);
/* model.hpp:95-124 (T, V = NmfModel::T[n_h], V[n_h]; K = rank) */
int rcscm_gpu_init_params(rcscm_gpu_ctx* ctx, const rcscm_inputs* in, int K,
                          const double* X, const double* W, const double* A,
                          const double* T, const double* V, rcscm_params* out);
/* model.hpp:129-157 */
int rcscm_gpu_map_objective(rcscm_gpu_ctx* ctx, const rcscm_inputs* in,
                            const rcscm_params* p, const rcscm_hyper* hyper,
                            const double* X, double* out);
/* solver_naive.hpp:412-450 */
int rcscm_gpu_run_naive(rcscm_gpu_ctx* ctx, const rcscm_inputs* in,
                        const rcscm_params* params0, const rcscm_hyper* hyper,
                        const double* X, const rcscm_solver_opts* opt,
                        rcscm_params* out, rcscm_result* extra);
/* solver_accel.hpp:245-250 (Algorithm 1: per-bin M x M inverse each iteration;
 * needs in->R_prime, not R_prime_pinv; complex128 in both context precisions) */
int rcscm_gpu_run_algorithm1(rcscm_gpu_ctx* ctx, const rcscm_inputs* in,
                             const rcscm_params* params0, const rcscm_hyper* hyper,
                             const double* X, const rcscm_solver_opts* opt,
                             rcscm_params* out, rcscm_result* extra);
/* solver_accel.hpp:254-258 */
int rcscm_gpu_run_algorithm2(rcscm_gpu_ctx* ctx, const rcscm_inputs* in,
                             const rcscm_params* params0, const rcscm_hyper* hyper,
                             const double* X, const rcscm_solver_opts* opt,
                             rcscm_params* out, rcscm_result* extra);
/* solver_accel.hpp:246-258 by stage: 1 = run_algorithm1, 2 = run_algorithm2 (the
 * accelerated entry as one symbol; any other stage is RCSCM_INVALID_INPUT). */
int rcscm_gpu_run_accel(rcscm_gpu_ctx* ctx, int stage, const rcscm_inputs* in,
                        const rcscm_params* params0, const rcscm_hyper* hyper,
                        const double* X, const rcscm_solver_opts* opt,
                        rcscm_params* out, rcscm_result* extra);
/* model.hpp:58-124 in one call: build_noise_scm (a, R', R'^+, b into the caller's
 * buffers, as rcscm_gpu_build_noise_scm) then init_params (params0 into out, T, V =
 * NmfModel::T[n_h], V[n_h], K = rank); the same results as the two calls. */
int rcscm_gpu_build_inputs(rcscm_gpu_ctx* ctx, int64_t I, int64_t J, int M,
                           const double* X, const double* W, const double* A,
                           int n_h, double rank_tol, int K, const double* T,
                           const double* V, double* a, double* R_prime,
                           double* R_prime_pinv, double* b, rcscm_params* out);
/* wiener.hpp:19-43 (image [i][t][m] and/or dry I x J col-major; either may be NULL) */
int rcscm_gpu_extract_target(rcscm_gpu_ctx* ctx, const rcscm_inputs* in,
                             const rcscm_params* p, const double* X, double* image,
                             double* dry);
/* wiener.hpp:46-53 */
int rcscm_gpu_extract_noise(rcscm_gpu_ctx* ctx, const rcscm_inputs* in,
                            const rcscm_params* p, const double* X, double* noise);

/* ---- STFT / ISTFT (the steps before and after the path) ------------------ */
/* stft.hpp:37-46 + :58-60: window / hop in samples, frame count
 * J = ceil((len + win - hop) / hop) and bin count win/2 + 1 (any output may be NULL) */
int rcscm_gpu_stft_shape(int64_t num_samples, double sample_rate, double win_ms,
                         double hop_ms, int* win, int* hop, int64_t* frames,
                         int64_t* bins);
/* stft.hpp:50-88: samples (M x len) -> X [i][t][m] (bins x frames x M) */
int rcscm_gpu_stft_analyze(rcscm_gpu_ctx* ctx, const double* samples,
                           int64_t num_samples, int M, double sample_rate,
                           double win_ms, double hop_ms, double* X);
/* stft.hpp:92-129: X [i][t][m] with the Spectrogram's win_samples / hop_samples /
 * source_samples -> samples (M x len), len = source_samples if > 0 else
 * J*hop - (win - hop) */
int rcscm_gpu_stft_synthesize(rcscm_gpu_ctx* ctx, const double* X, int64_t I,
                              int64_t J, int M, double sample_rate, int spec_win,
                              int spec_hop, int64_t source_samples, double win_ms,
                              double hop_ms, double* samples);

/* ---- sphering + ILRMA (the step before the path) --------------------------- */
/* ilrma.hpp:53-73: X [i][t][m] -> Q (whitening, [i][M*M]) and Q X; either output may be NULL */
int rcscm_gpu_sphere(rcscm_gpu_ctx* ctx, int64_t I, int64_t J, int M, const double* X,
                     double* Q, double* Xw);
/* ilrma.hpp:145-240: Gaussian ILRMA on (whitened) X [i][t][m] with K NMF bases
 * (K <= 16), iters IP + NMF sweeps and the reference's seeded initialisation.
 * Outputs (any may be NULL): W, A [i][M*M]; T [n] I x K col-major; V [n] K x J col-major. */
int rcscm_gpu_run_ilrma(rcscm_gpu_ctx* ctx, int64_t I, int64_t J, int M, int K,
                        int iters, uint64_t seed, const double* X, double* W, double* A,
                        double* T, double* V);

/* ---- cmd_extract on the device (tools/rcscm.cpp:158-221) ------------------
 * STFT -> sphering -> ILRMA -> fold (W = W_ilrma Q, A = W^{-1}) -> target index
 * (select_target_index when target_index < 0) -> build_noise_scm -> init_params
 * -> solver (backend 0 naive, 1 Algorithm 1, 2 Algorithm 2; optional objective
 * per iteration with the rel_obj_tol early stop) -> extract_target / extract_noise
 * -> WOLA synthesis, with every intermediate resident in HBM. samples, target and
 * noise are M x num_samples col-major (Waveform::samples) or channel rows
 * (samples_layout); target / noise may be NULL. */
typedef struct {
  double sample_rate, win_ms, hop_ms; /* 16000, 64, 32 in cmd_extract */
  int nmf_bases, ilrma_iters;         /* RunConfig defaults 10, 50 */
  uint64_t seed;
  int target_index;                   /* < 0: select_target_index */
  int backend;                        /* 0 naive, 1 accel1, 2 accel2 */
  int iters;
  double alpha, beta, eps_var, rel_obj_tol;
  int compute_objective;              /* cmd_extract sets it */
  int samples_layout;                 /* 0: samples / target / noise M x num_samples col-major
                                         (Waveform::samples); 1: one contiguous row of
                                         num_samples per channel (numpy (M, n) C order) */
} rcscm_extract_opts;
typedef struct {
  int target_index, n_iters;
  int64_t bins, frames;
  double* objective;                  /* caller buffer, >= iters + 1 entries, or NULL */
  int n_objective;
  double* iter_seconds;               /* caller buffer, >= iters entries, or NULL: CUDA-event
                                         time of each solver iteration, objective excluded
                                         (solver_accel.hpp:205,227); without compute_objective
                                         the iterations run as one launch and share its time */
} rcscm_extract_result;
int rcscm_gpu_extract(rcscm_gpu_ctx* ctx, const rcscm_extract_opts* opts,
                      const double* samples, int64_t num_samples, int M,
                      double* target, double* noise, rcscm_extract_result* result);

/* ---- device-resident session (bench / pipelines) -------------------------
 * A session keeps one problem (B utterances x I bins x J frames x M mics,
 * bins flattened utterance-major) resident in HBM in the device layout, so a
 * pipeline step can be timed with its inputs already on the GPU.
 * X: [u][i][t][m]; W, A: [u][i] M x M col-major; T: [u] I x K col-major;
 * V: [u] K x J col-major. Launches are asynchronous on the context stream. */
int rcscm_gpu_session_load(rcscm_gpu_ctx* ctx, int64_t B, int64_t I, int64_t J,
                           int M, int K, int n_h, const double* X, const double* W,
                           const double* A, const double* T, const double* V);
/* Stage flags for rcscm_gpu_session_run */
#define RCSCM_STAGE_SETUP 1     /* build_noise_scm + init_params (from X, W, A, T, V) */
#define RCSCM_STAGE_PRECOMPUTE 2 /* sigma / tau (solver_accel.hpp:33-64) */
#define RCSCM_STAGE_ACCEL 4     /* Algorithm 2 iterations (on-chip kernel) */
#define RCSCM_STAGE_NAIVE 8     /* naive EM iterations */
#define RCSCM_STAGE_WIENER 16   /* extract_target from the resident state */
#define RCSCM_STAGE_RESET 32    /* restore params0 (from the last SETUP) before iterating */
int rcscm_gpu_session_run(rcscm_gpu_ctx* ctx, int stages, int iters,
                          const rcscm_hyper* hyper, double eps_var);
/* Asynchronous copy of the session outputs (any pointer may be NULL) into host
 * or device memory of this context's device (unified addressing picks the
 * direction; a multi-GPU caller fetches into its transfer buffers for the
 * gather); synchronizes the stream before returning when sync != 0.
 * Layouts: r_h, r_u [u][i][t]; lambda [u][i]; dry [u][i][t] complex;
 * image [u][i][t][m] complex. */
int rcscm_gpu_session_fetch(rcscm_gpu_ctx* ctx, double* r_h, double* r_u,
                            double* lambda, double* dry, double* image, int sync);
/* Last RCSCM_STAGE_* error raised on the device (0 if none); synchronizes. */
int rcscm_gpu_session_check(rcscm_gpu_ctx* ctx);
/* The stream the context launches on (cudaStream_t as void*). */
void* rcscm_gpu_stream(rcscm_gpu_ctx* ctx);

/* ---- diagnostics ----------------------------------------------------------
 * Measured FP64 FMA-pipe throughput of this device (independent DFMA chains on
 * every SM), the denominator of the accel kernel's roofline fraction. */
int rcscm_gpu_probe_fp64(rcscm_gpu_ctx* ctx, double* tflops, double* ms);
/* Same for the FP32 FMA pipe (denominator of the complex64 mode). */
int rcscm_gpu_probe_fp32(rcscm_gpu_ctx* ctx, double* tflops, double* ms);

#ifdef __cplusplus
}
#endif
#endif /* RCSCM_GPU_H */
