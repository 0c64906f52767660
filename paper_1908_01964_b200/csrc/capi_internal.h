// capi_internal.h -- shared internals of the C ABI translation units (capi.cu:
// the reference entry points, solvers and session; capi_pipeline.cu: STFT,
// sphering, ILRMA and the device cmd_extract chain). Not a public header.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../../include/rcscm_gpu.h"
#include "launch.h"

using namespace rcscm;

namespace rcscm_capi {

extern thread_local std::string g_last_error;

struct ApiError {
  int code;
  std::string msg;
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw ApiError{code, msg}; }

#define CK(expr)                                                                                      \
  do {                                                                                                \
    cudaError_t e_ = (expr);                                                                          \
    if (e_ != cudaSuccess) fail(RCSCM_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// Grow-only device buffer.
struct DBuf {
  void* p = nullptr;
  size_t cap = 0;
  template <class T>
  T* get(size_t n) {
    const size_t bytes = std::max<size_t>(n * sizeof(T), 16);
    if (bytes > cap) {
      if (p) cudaFree(p);
      p = nullptr;
      cap = 0;
      CK(cudaMalloc(&p, bytes));
      cap = bytes;
    }
    return static_cast<T*>(p);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// Page-locked host staging (grown on demand): waveform copies at full DMA rate
// instead of the driver's pageable path.
struct HBuf {
  void* p = nullptr;
  size_t cap = 0;
  template <class T>
  T* get(size_t n) {
    const size_t bytes = std::max<size_t>(n * sizeof(T), 16);
    if (bytes > cap) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      cap = 0;
      CK(cudaMallocHost(&p, bytes));
      cap = bytes;
    }
    return static_cast<T*>(p);
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
};

constexpr int kMaxChunks = 16;
constexpr double kEpsVar = 1e-12;  // types.hpp:55 (init_params' floor)

inline void check_mics(int M) {
  if (!mics_supported(M)) fail(RCSCM_UNSUPPORTED, "mics = " + std::to_string(M) + " is not supported (1..16)");
}

}  // namespace rcscm_capi

using rcscm_capi::DBuf;
using rcscm_capi::HBuf;
using rcscm_capi::fail;

struct rcscm_gpu_ctx {
  int device = 0;
  int precision = RCSCM_C128;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int64_t launches = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // two copy streams (one DMA engine each: a single H2D stream reaches half the
  // PCIe rate on B200 hosts) and a compute stream for the pipelined entry points
  cudaStream_t aux[4] = {nullptr, nullptr, nullptr, nullptr};  // + a D2H stream
  cudaEvent_t evx[22] = {};  // kMaxChunks + 6
  cudaEvent_t evt[32] = {};  // 2 * kMaxChunks timing events: each pipelined chunk's K2 launch
  // device buffers
  DBuf X, W, A, T, V, a, b, Rp, Rpp, power, sab, taa, sbx, tax, txx, rh, ru, lam, lpd;
  DBuf rh0, ru0, lam0, tmp, tmp2, traj_rh, traj_ru, traj_lam, scratch, dry, image, noise, partial, obj, err;
  DBuf gam;  // Algorithm 1 scratch (gamma per slot)
  DBuf obj_part;  // K2's per-iteration, per-CTA objective partials
  DBuf st_part, st_lam;  // streaming Algorithm 2 (bins > on-chip capacity): chunk partials, lambda ping-pong
  // STFT: waveform, window table, frames, half spectra, Spectrogram
  DBuf st_x, st_w, st_f, st_spec, st_X;
  // ILRMA: whitened x, W, A, T, V, powers, partial sums, mu
  DBuf il_X, il_W, il_A, il_T, il_V, il_P, il_part, il_mu, il_Pt, il_ucov;
  // extract pipeline: whitening Q, folded W / A, target powers, output waveform,
  // objective trace
  DBuf ex_Q, ex_W, ex_A, ex_pow, ex_out, ex_obj;
  HBuf ex_pin;  // pinned staging of the waveforms in and out
  HBuf err_pin;  // pinned landing word of the device error word (check_err)
  StftPlan stft_plan;
  // ILRMA sweeps replayed as one CUDA graph, re-captured when the shape, the
  // buffers or the sweep count change (key: IlrmaArgs fields, M, iters)
  cudaGraphExec_t il_graph = nullptr;
  std::vector<int64_t> il_graph_key;
  int il_graph_launches = 0;
  // complex64 (FP32) mode copies of the slot arrays
  DBuf Xf, sbxf, taxf, txxf, rhf, ruf, dryf, imagef, rh0f, ru0f;
  bool f32_params_current = false;  // session: FP32 r_h / r_u hold the latest iterate
  // session geometry
  bool s_loaded = false, s_setup = false, s_pre = false;
  // RESET is applied lazily: the next ACCEL reads params0 directly (no copy
  // pass); any other consumer of the iterate materialises it first.
  bool s_reset_pending = false;
  int64_t sB = 0, sI = 0, sJ = 0;
  int sM = 0, sK = 0, sn_h = 0;
  // multi-device: the contexts of devices[1..] (this one is devices[0]); while a
  // context serves one bin range of a sharded call, ldh is the caller's I (the
  // leading dimension of its I x J col-major host arrays) and bin_offset the
  // range's first bin (error messages report global bins)
  std::vector<rcscm_gpu_ctx*> peers;
  int64_t ldh = 0, bin_offset = 0;

  // Every kernel launch goes through here: the error is surfaced as
  // RCSCM_CUDA_ERROR and the launch counter (rcscm_gpu_launch_count) advances.
  void launched(cudaError_t e, int n = 1) {
    if (e != cudaSuccess) fail(RCSCM_CUDA_ERROR, std::string("kernel launch: ") + cudaGetErrorString(e));
    launches += n;
  }
};

namespace rcscm_capi {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return RCSCM_OK;
  } catch (const ApiError& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return RCSCM_CUDA_ERROR;
  }
}


// helpers defined in capi.cu
void h2d(rcscm_gpu_ctx* c, void* dst, const void* src, size_t bytes);
void d2h(rcscm_gpu_ctx* c, void* dst, const void* src, size_t bytes);
void d2d(rcscm_gpu_ctx* c, void* dst, const void* src, size_t bytes);
// I x J col-major host array (leading dimension c->ldh when serving a bin range
// of a wider array) <-> contiguous I x J device array, element size esz
void h2d_ij(rcscm_gpu_ctx* c, void* dst, const void* src, int64_t I, int64_t J, size_t esz);
void d2h_ij(rcscm_gpu_ctx* c, void* dst, const void* src, int64_t I, int64_t J, size_t esz);
void sync(rcscm_gpu_ctx* c);
void reset_err(rcscm_gpu_ctx* c);
void check_err(rcscm_gpu_ctx* c, int64_t J);
DevProblem problem(rcscm_gpu_ctx* c, int64_t B, int64_t I, int64_t J, int M);
bool f32(const rcscm_gpu_ctx* c);
void params_from_f32(rcscm_gpu_ctx* c, size_t S);
Accel1Args accel1_args(rcscm_gpu_ctx* c, int64_t nb, int64_t J, int iters, const rcscm_hyper& h, double eps,
                       double gamma_fault);
// MAP objective (dev_out: leave the value in that device slot, no host round trip)
double objective(rcscm_gpu_ctx* c, int64_t nb, int64_t J, int M, const rcscm_hyper& h, double* dev_out = nullptr);
double objective_fast(rcscm_gpu_ctx* c, int64_t nb, int64_t J, int M, const rcscm_hyper& h,
                      double* dev_out = nullptr);
// Algorithm 2 for `iters` iterations with the objective after each iteration
// evaluated inside K2 into dobj[1..iters] (dobj[0]: the caller's initial value);
// optional trajectory buffers ([it][bin][t], [it][bin]). One K2 launch + one
// row reduction; complex128 only.
void run_accel_obj(rcscm_gpu_ctx* c, int64_t I, int64_t J, int M, int iters, const rcscm_hyper& h, double eps,
                   double gamma_fault, double* dobj, double* trh = nullptr, double* tru = nullptr,
                   double* trl = nullptr);
// session_load from host (H2D) or device (D2D) buffers
void session_load_impl(rcscm_gpu_ctx* c, int64_t B, int64_t I, int64_t J, int M, int K, int n_h, const void* X,
                       const void* W, const void* A, const void* T, const void* V, cudaMemcpyKind kind);

}  // namespace rcscm_capi
