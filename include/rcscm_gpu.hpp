// rcscm_gpu.hpp -- header-only C++17 front end of the C ABI (rcscm_gpu.h) with
// the reference's entry-point names, argument meaning and exceptions:
//
//   rcscm::gpu::build_noise_scm   <- rcscm::build_noise_scm   model.hpp:58-90
//   rcscm::gpu::init_params       <- rcscm::init_params       model.hpp:95-124
//   rcscm::gpu::map_objective     <- rcscm::map_objective     model.hpp:129-157
//   rcscm::gpu::run_naive         <- rcscm::run_naive         solver_naive.hpp:412-450
//   rcscm::gpu::run_algorithm1    <- rcscm::run_algorithm1    solver_accel.hpp:245-250
//   rcscm::gpu::run_algorithm2    <- rcscm::run_algorithm2    solver_accel.hpp:254-258
//   rcscm::gpu::extract_target    <- rcscm::extract_target    wiener.hpp:19-43
//   rcscm::gpu::extract_noise     <- rcscm::extract_noise     wiener.hpp:46-53
//   rcscm::gpu::stft_analyze      <- rcscm::stft_analyze      stft.hpp:50-88
//   rcscm::gpu::stft_synthesize   <- rcscm::stft_synthesize   stft.hpp:92-129
//
// The containers below are plain std::vector stand-ins with the reference's
// Eigen column-major layouts (see rcscm_gpu.h), so a caller holding Eigen
// matrices can pass .data() pointers without copying (INTEGRATION.md shows the
// adapter for the reference's own RcscmInputs / RcscmParams / Spectrogram).
// Failures throw InvalidInputError / NumericalError exactly where the
// reference throws (types.hpp:20-30); CUDA failures throw CudaError.
#pragma once

#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "rcscm_gpu.h"

namespace rcscm {
namespace gpu {

using cplx = std::complex<double>;

struct InvalidInputError : std::invalid_argument {
  explicit InvalidInputError(const std::string& w) : std::invalid_argument(w) {}
};
struct NumericalError : std::runtime_error {
  explicit NumericalError(const std::string& w) : std::runtime_error(w) {}
};
struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};

inline void check(int rc) {
  if (rc == RCSCM_OK) return;
  const std::string msg = rcscm_gpu_last_error();
  if (rc == RCSCM_INVALID_INPUT) throw InvalidInputError(msg);
  if (rc == RCSCM_NUMERICAL) throw NumericalError(msg);
  throw CudaError(msg);
}

// types.hpp:43-53: bins[i] is M x J col-major -> data[(i*J + t)*M + m]; the
// STFT metadata travel with it as in the reference
struct Spectrogram {
  int64_t bins = 0, frames = 0;
  int mics = 0;
  std::vector<cplx> data;
  double sample_rate = 16000.0;
  int win_samples = 0, hop_samples = 0;
  int64_t source_samples = 0;
  const double* ptr() const { return reinterpret_cast<const double*>(data.data()); }
};

// types.hpp:33-39: samples is channels x num_samples col-major -> data[ch + p*M]
struct Waveform {
  int channels = 0;
  int64_t num_samples = 0;
  std::vector<double> samples;
  double sample_rate = 16000.0;
};

// model.hpp:16-25
struct RcscmInputs {
  int64_t bins = 0;
  int mics = 0;
  int n_h = 0;
  std::vector<cplx> a, b;                   // [i][m]
  std::vector<cplx> R_prime, R_prime_pinv;  // [i][r + c*M]
};

// model.hpp:29-33 (r_h / r_u: element (i, t) at i + t*I)
struct RcscmParams {
  int64_t bins = 0, frames = 0;
  std::vector<double> r_h, r_u, lambda;
};

struct Hyperparams {  // model.hpp:36-39
  double alpha = 1.1;
  double beta = 1e-16;
};

struct SolverOptions {  // solver_naive.hpp:14-22
  int iters = 200;
  bool compute_objective = false;
  bool record_trajectory = false;
  double rel_obj_tol = 0.0;
  int threads = 1;
  double eps_var = 1e-12;
  double gamma_fault = 0.0;
};

struct SolverResult {  // solver_naive.hpp:24-29
  RcscmParams params;
  std::vector<double> objective, iter_seconds;
  std::vector<RcscmParams> trajectory;
};

struct ExtractionResult {  // wiener.hpp:11-14
  Spectrogram image;
  std::vector<cplx> dry;  // (i, t) at i + t*I
};

// One CUDA device + stream (rcscm_gpu_ctx), or bins sharded over a device list
// (one stream and host thread per device). Not thread-safe; one per thread.
class Context {
 public:
  explicit Context(int device = 0, void* stream = nullptr) {
    rcscm_gpu_config cfg{device, RCSCM_C128, stream, nullptr, 0};
    check(rcscm_gpu_create(&cfg, &ctx_));
  }
  explicit Context(const std::vector<int>& devices) {
    rcscm_gpu_config cfg{devices.empty() ? 0 : devices[0], RCSCM_C128, nullptr, devices.data(),
                         static_cast<int>(devices.size())};
    check(rcscm_gpu_create(&cfg, &ctx_));
  }
  ~Context() { rcscm_gpu_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  rcscm_gpu_ctx* get() const { return ctx_; }

 private:
  rcscm_gpu_ctx* ctx_ = nullptr;
};

namespace detail {
inline rcscm_inputs view(const RcscmInputs& in, int64_t frames) {
  rcscm_inputs v{};
  v.num_bins = in.bins;
  v.frames = frames;
  v.mics = in.mics;
  v.n_h = in.n_h;
  v.a = reinterpret_cast<const double*>(in.a.data());
  v.b = reinterpret_cast<const double*>(in.b.data());
  v.R_prime = in.R_prime.empty() ? nullptr : reinterpret_cast<const double*>(in.R_prime.data());
  v.R_prime_pinv = in.R_prime_pinv.empty() ? nullptr : reinterpret_cast<const double*>(in.R_prime_pinv.data());
  return v;
}
inline RcscmParams alloc_params(int64_t I, int64_t J) {
  RcscmParams p;
  p.bins = I;
  p.frames = J;
  p.r_h.assign(I * J, 0.0);
  p.r_u.assign(I * J, 0.0);
  p.lambda.assign(I, 0.0);
  return p;
}
// backend: 0 = run_naive, 1 = run_algorithm1, 2 = run_algorithm2
inline SolverResult run(Context& ctx, int backend, const RcscmInputs& in, const RcscmParams& p0,
                        const Hyperparams& hyper, const Spectrogram& X, const SolverOptions& opt) {
  const int64_t I = in.bins, J = X.frames;
  const rcscm_inputs v = view(in, J);
  rcscm_params pin{const_cast<double*>(p0.r_h.data()), const_cast<double*>(p0.r_u.data()),
                   const_cast<double*>(p0.lambda.data())};
  const rcscm_hyper h{hyper.alpha, hyper.beta};
  const rcscm_solver_opts o{opt.iters, opt.compute_objective, opt.record_trajectory, opt.rel_obj_tol,
                            opt.threads, opt.eps_var, opt.gamma_fault};
  SolverResult res;
  res.params = alloc_params(I, J);
  rcscm_params pout{res.params.r_h.data(), res.params.r_u.data(), res.params.lambda.data()};
  const int n = opt.iters > 0 ? opt.iters : 0;
  res.objective.assign(n + 1, 0.0);
  res.iter_seconds.assign(n, 0.0);
  std::vector<double> th, tu, tl;
  if (opt.record_trajectory) {
    th.assign(static_cast<size_t>(n) * I * J, 0.0);
    tu.assign(static_cast<size_t>(n) * I * J, 0.0);
    tl.assign(static_cast<size_t>(n) * I, 0.0);
  }
  int n_obj = 0, n_it = 0;
  rcscm_result extra{res.objective.data(), &n_obj, res.iter_seconds.data(), &n_it,
                     opt.record_trajectory ? th.data() : nullptr, opt.record_trajectory ? tu.data() : nullptr,
                     opt.record_trajectory ? tl.data() : nullptr};
  check(backend == 2   ? rcscm_gpu_run_algorithm2(ctx.get(), &v, &pin, &h, X.ptr(), &o, &pout, &extra)
        : backend == 1 ? rcscm_gpu_run_algorithm1(ctx.get(), &v, &pin, &h, X.ptr(), &o, &pout, &extra)
                       : rcscm_gpu_run_naive(ctx.get(), &v, &pin, &h, X.ptr(), &o, &pout, &extra));
  res.objective.resize(n_obj);
  res.iter_seconds.resize(n_it);
  for (int k = 0; opt.record_trajectory && k < n_it; ++k) {
    RcscmParams s = alloc_params(I, J);
    std::copy(th.begin() + k * I * J, th.begin() + (k + 1) * I * J, s.r_h.begin());
    std::copy(tu.begin() + k * I * J, tu.begin() + (k + 1) * I * J, s.r_u.begin());
    std::copy(tl.begin() + k * I, tl.begin() + (k + 1) * I, s.lambda.begin());
    res.trajectory.push_back(std::move(s));
  }
  return res;
}
}  // namespace detail

// W, A: per bin M x M col-major ([i][r + c*M]), as DemixingSet (ilrma.hpp:19-22).
inline RcscmInputs build_noise_scm(Context& ctx, const std::vector<cplx>& W, const std::vector<cplx>& A,
                                   const Spectrogram& X, int n_h, double rank_tol = 1e-10) {
  RcscmInputs in;
  in.bins = X.bins;
  in.mics = X.mics;
  in.n_h = n_h;
  const size_t I = X.bins, M = X.mics;
  in.a.assign(I * M, 0.0);
  in.b.assign(I * M, 0.0);
  in.R_prime.assign(I * M * M, 0.0);
  in.R_prime_pinv.assign(I * M * M, 0.0);
  auto d = [](std::vector<cplx>& v) { return reinterpret_cast<double*>(v.data()); };
  check(rcscm_gpu_build_noise_scm(ctx.get(), X.bins, X.frames, X.mics, X.ptr(),
                                  reinterpret_cast<const double*>(W.data()),
                                  reinterpret_cast<const double*>(A.data()), n_h, rank_tol, d(in.a),
                                  d(in.R_prime), d(in.R_prime_pinv), d(in.b)));
  return in;
}

// T = NmfModel::T[n_h] (I x K col-major), V = NmfModel::V[n_h] (K x J col-major).
inline RcscmParams init_params(Context& ctx, const RcscmInputs& in, const std::vector<double>& T,
                               const std::vector<double>& V, int K, const std::vector<cplx>& W,
                               const std::vector<cplx>& A, const Spectrogram& X) {
  RcscmParams p = detail::alloc_params(in.bins, X.frames);
  const rcscm_inputs v = detail::view(in, X.frames);
  rcscm_params out{p.r_h.data(), p.r_u.data(), p.lambda.data()};
  check(rcscm_gpu_init_params(ctx.get(), &v, K, X.ptr(), reinterpret_cast<const double*>(W.data()),
                              reinterpret_cast<const double*>(A.data()), T.data(), V.data(), &out));
  return p;
}

inline double map_objective(Context& ctx, const RcscmInputs& in, const RcscmParams& p, const Hyperparams& hyper,
                            const Spectrogram& X) {
  const rcscm_inputs v = detail::view(in, X.frames);
  rcscm_params pv{const_cast<double*>(p.r_h.data()), const_cast<double*>(p.r_u.data()),
                  const_cast<double*>(p.lambda.data())};
  const rcscm_hyper h{hyper.alpha, hyper.beta};
  double out = 0.0;
  check(rcscm_gpu_map_objective(ctx.get(), &v, &pv, &h, X.ptr(), &out));
  return out;
}

inline SolverResult run_naive(Context& ctx, const RcscmInputs& in, const RcscmParams& params0,
                              const Hyperparams& hyper, const Spectrogram& X, const SolverOptions& opt) {
  return detail::run(ctx, 0, in, params0, hyper, X, opt);
}

inline SolverResult run_algorithm1(Context& ctx, const RcscmInputs& in, const RcscmParams& params0,
                                   const Hyperparams& hyper, const Spectrogram& X, const SolverOptions& opt) {
  return detail::run(ctx, 1, in, params0, hyper, X, opt);
}

inline SolverResult run_algorithm2(Context& ctx, const RcscmInputs& in, const RcscmParams& params0,
                                   const Hyperparams& hyper, const Spectrogram& X, const SolverOptions& opt) {
  return detail::run(ctx, 2, in, params0, hyper, X, opt);
}

inline ExtractionResult extract_target(Context& ctx, const RcscmInputs& in, const RcscmParams& p,
                                       const Spectrogram& X) {
  ExtractionResult out;
  out.image = X;
  out.dry.assign(static_cast<size_t>(X.bins * X.frames), 0.0);
  const rcscm_inputs v = detail::view(in, X.frames);
  rcscm_params pv{const_cast<double*>(p.r_h.data()), const_cast<double*>(p.r_u.data()),
                  const_cast<double*>(p.lambda.data())};
  check(rcscm_gpu_extract_target(ctx.get(), &v, &pv, X.ptr(), reinterpret_cast<double*>(out.image.data.data()),
                                 reinterpret_cast<double*>(out.dry.data())));
  return out;
}

inline Spectrogram extract_noise(Context& ctx, const RcscmInputs& in, const RcscmParams& p, const Spectrogram& X) {
  Spectrogram noise = X;
  const rcscm_inputs v = detail::view(in, X.frames);
  rcscm_params pv{const_cast<double*>(p.r_h.data()), const_cast<double*>(p.r_u.data()),
                  const_cast<double*>(p.lambda.data())};
  check(rcscm_gpu_extract_noise(ctx.get(), &v, &pv, X.ptr(), reinterpret_cast<double*>(noise.data.data())));
  return noise;
}

inline Spectrogram stft_analyze(Context& ctx, const Waveform& w, double win_ms, double hop_ms) {
  int win = 0, hop = 0;
  int64_t J = 0, B = 0;
  check(rcscm_gpu_stft_shape(w.num_samples, w.sample_rate, win_ms, hop_ms, &win, &hop, &J, &B));
  Spectrogram s;
  s.bins = B;
  s.frames = J;
  s.mics = w.channels;
  s.sample_rate = w.sample_rate;
  s.win_samples = win;
  s.hop_samples = hop;
  s.source_samples = w.num_samples;
  s.data.assign(static_cast<size_t>(B * J) * (w.channels > 0 ? w.channels : 0), cplx(0.0, 0.0));
  check(rcscm_gpu_stft_analyze(ctx.get(), w.samples.data(), w.num_samples, w.channels, w.sample_rate, win_ms, hop_ms,
                               reinterpret_cast<double*>(s.data.data())));
  return s;
}

inline Waveform stft_synthesize(Context& ctx, const Spectrogram& s, double win_ms, double hop_ms) {
  Waveform w;
  w.channels = s.mics;
  w.sample_rate = s.sample_rate;
  const int64_t len = s.source_samples > 0 ? s.source_samples
                                           : s.frames * s.hop_samples - (s.win_samples - s.hop_samples);
  w.num_samples = len > 0 ? len : 0;
  w.samples.assign(static_cast<size_t>(w.num_samples) * (s.mics > 0 ? s.mics : 0), 0.0);
  check(rcscm_gpu_stft_synthesize(ctx.get(), s.ptr(), s.bins, s.frames, s.mics, s.sample_rate, s.win_samples,
                                  s.hop_samples, s.source_samples, win_ms, hop_ms, w.samples.data()));
  return w;
}

}  // namespace gpu
}  // namespace rcscm
