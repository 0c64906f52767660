// capi_pipeline.cu -- C ABI of the steps around the SCM path (include/rcscm_gpu.h):
// STFT analysis / WOLA synthesis (stft.hpp), sphering and ILRMA (ilrma.hpp) and
// the whole cmd_extract chain on the device (tools/rcscm.cpp:158-221). Kernels:
// stft.cu, ilrma.cu; the SCM stages reuse the session of capi.cu.
#include <thread>

#include "capi_internal.h"

using namespace rcscm_capi;

namespace {

// Replays the ~7 (iters + 5) launches of the ILRMA sweeps as one CUDA graph:
// launch overhead, not kernel time, dominated them at the reference's sizes.
template <typename F>
static void ilrma_graph_launch(rcscm_gpu_ctx* c, const IlrmaArgs& a, int M, int iters, F&& sweeps) {
  const std::vector<int64_t> key{a.I, a.J, a.K, M, iters, reinterpret_cast<int64_t>(a.X),
                                 reinterpret_cast<int64_t>(a.W), reinterpret_cast<int64_t>(a.A),
                                 reinterpret_cast<int64_t>(a.T), reinterpret_cast<int64_t>(a.V),
                                 reinterpret_cast<int64_t>(a.P), reinterpret_cast<int64_t>(a.Pt),
                                 reinterpret_cast<int64_t>(a.partial), reinterpret_cast<int64_t>(a.mu),
                                 reinterpret_cast<int64_t>(a.ucov), reinterpret_cast<int64_t>(a.err)};
  if (!c->il_graph || key != c->il_graph_key) {
    if (c->il_graph) cudaGraphExecDestroy(c->il_graph);
    c->il_graph = nullptr;
    const int64_t before = c->launches;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    cudaGraph_t g = nullptr;
    try {
      sweeps();
    } catch (...) {
      cudaStreamEndCapture(c->stream, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    CK(cudaStreamEndCapture(c->stream, &g));
    const cudaError_t ie = cudaGraphInstantiate(&c->il_graph, g, 0);
    cudaGraphDestroy(g);
    CK(ie);
    c->il_graph_key = key;
    c->il_graph_launches = static_cast<int>(c->launches - before);
  } else {
    c->launches += c->il_graph_launches;
  }
  CK(cudaGraphLaunch(c->il_graph, c->stream));
}

}  // namespace

extern "C" {

// ---- STFT / ISTFT (stft.hpp) ------------------------------------------------------
// detail::stft_params (stft.hpp:37-46) and the frame count of stft_analyze (:58-60)
static void stft_params(double sample_rate, double win_ms, double hop_ms, int* win, int* hop) {
  if (!(win_ms > hop_ms && hop_ms > 0)) fail(RCSCM_INVALID_INPUT, "stft: require win_ms > hop_ms > 0");
  *win = static_cast<int>(std::lround(win_ms * 1e-3 * sample_rate));
  *hop = static_cast<int>(std::lround(hop_ms * 1e-3 * sample_rate));
  if (*win < 2 || *hop < 1) fail(RCSCM_INVALID_INPUT, "stft: window shorter than 2 samples");
}

// stft.hpp:12-17 periodic Hamming window, evaluated exactly as the reference
static std::vector<double> hamming(int n) {
  std::vector<double> w(n);
  for (int k = 0; k < n; ++k) w[k] = 0.54 - 0.46 * std::cos(2.0 * M_PI * k / n);
  return w;
}

int rcscm_gpu_stft_shape(int64_t num_samples, double sample_rate, double win_ms, double hop_ms, int* win, int* hop,
                         int64_t* frames, int64_t* bins) {
  return guarded([&] {
    int w = 0, h = 0;
    stft_params(sample_rate, win_ms, hop_ms, &w, &h);
    if (win) *win = w;
    if (hop) *hop = h;
    if (frames) *frames = (num_samples + (w - h) + h - 1) / h;
    if (bins) *bins = w / 2 + 1;
  });
}

// device STFT of the device waveform dx (M x len) into c->st_X ([bin][frame][mic])
static void stft_analyze_dev(rcscm_gpu_ctx* c, const double* dx, int64_t len, int M, double sample_rate,
                             double win_ms, double hop_ms, int* win_o, int* hop_o, int64_t* J_o, int64_t* B_o,
                             bool planar = false) {
  int win = 0, hop = 0;
  stft_params(sample_rate, win_ms, hop_ms, &win, &hop);
  const int64_t J = (len + (win - hop) + hop - 1) / hop, B = win / 2 + 1, rows = J * M;
  const std::vector<double> w = hamming(win);
  double* dw = c->st_w.get<double>(win);
  h2d(c, dw, w.data(), win * sizeof(double));
  double2* dX = c->st_X.get<double2>(static_cast<size_t>(B * rows));
  c->launched(launch_stft_analyze(c->stream, c->stft_plan, dx, len, M, win, hop, J, dw,
                                  c->st_f.get<double>(static_cast<size_t>(rows) * win),
                                  c->st_spec.get<double2>(static_cast<size_t>(rows * B)), dX, planar),
              3);
  *win_o = win;
  *hop_o = hop;
  *J_o = J;
  *B_o = B;
}

// device WOLA synthesis of dX ([bin][frame][mic], I = win/2 + 1 bins) into dout (M x len)
static void stft_synth_dev(rcscm_gpu_ctx* c, const double2* dX, int64_t I, int64_t J, int M, int win, int hop,
                           int64_t len, double* dout, bool planar = false) {
  const std::vector<double> w = hamming(win);
  std::vector<double> denom(hop, 0.0), dual(win);
  for (int k = 0; k < win; ++k) denom[k % hop] += w[k] * w[k];
  for (int k = 0; k < win; ++k) dual[k] = (w[k] / denom[k % hop]) / win;  // wola_dual_window / win
  double* dd = c->st_w.get<double>(win);
  h2d(c, dd, dual.data(), win * sizeof(double));
  const int64_t rows = J * M;
  c->launched(launch_stft_synthesize(c->stream, c->stft_plan, dX, I, J, M, win, hop, len, dd,
                                     c->st_spec.get<double2>(static_cast<size_t>(rows * I)),
                                     c->st_f.get<double>(static_cast<size_t>(rows) * win), dout, planar),
              4);
}

int rcscm_gpu_stft_analyze(rcscm_gpu_ctx* c, const double* samples, int64_t num_samples, int M, double sample_rate,
                           double win_ms, double hop_ms, double* X) {
  return guarded([&] {
    if (!c) fail(RCSCM_INVALID_INPUT, "ctx must not be NULL");
    if (num_samples <= 0 || M <= 0) fail(RCSCM_INVALID_INPUT, "stft_analyze: empty waveform");
    if (!samples || !X) fail(RCSCM_INVALID_INPUT, "stft_analyze: NULL buffer");
    int win = 0, hop = 0;
    stft_params(sample_rate, win_ms, hop_ms, &win, &hop);
    double* dx = c->st_x.get<double>(static_cast<size_t>(num_samples) * M);
    h2d(c, dx, samples, static_cast<size_t>(num_samples) * M * sizeof(double));
    int64_t J = 0, B = 0;
    stft_analyze_dev(c, dx, num_samples, M, sample_rate, win_ms, hop_ms, &win, &hop, &J, &B);
    d2h(c, X, c->st_X.p, static_cast<size_t>(B * J * M) * sizeof(double2));
    sync(c);
  });
}

int rcscm_gpu_stft_synthesize(rcscm_gpu_ctx* c, const double* X, int64_t I, int64_t J, int M, double sample_rate,
                              int spec_win, int spec_hop, int64_t source_samples, double win_ms, double hop_ms,
                              double* samples) {
  return guarded([&] {
    if (!c) fail(RCSCM_INVALID_INPUT, "ctx must not be NULL");
    if (I <= 0) fail(RCSCM_INVALID_INPUT, "stft_synthesize: empty spectrogram");
    int win = 0, hop = 0;
    stft_params(sample_rate, win_ms, hop_ms, &win, &hop);
    if (win != spec_win || hop != spec_hop)
      fail(RCSCM_INVALID_INPUT, "stft_synthesize: window/hop do not match analysis");
    if (I != win / 2 + 1) fail(RCSCM_INVALID_INPUT, "stft_synthesize: bin count inconsistent with window");
    const int64_t pad = win - hop;
    const int64_t len = source_samples > 0 ? source_samples : J * hop - pad;
    if (len <= 0 || M <= 0 || J <= 0) fail(RCSCM_INVALID_INPUT, "stft_synthesize: empty spectrogram");
    if (!X || !samples) fail(RCSCM_INVALID_INPUT, "stft_synthesize: NULL buffer");
    const int64_t rows = J * M;
    double2* dX = c->st_X.get<double2>(static_cast<size_t>(I * rows));
    h2d(c, dX, X, static_cast<size_t>(I * rows) * sizeof(double2));
    double* dout = c->st_x.get<double>(static_cast<size_t>(len) * M);
    stft_synth_dev(c, dX, I, J, M, win, hop, len, dout);
    d2h(c, samples, dout, static_cast<size_t>(len) * M * sizeof(double));
    sync(c);
  });
}

// ---- sphering + ILRMA (ilrma.hpp) ----------------------------------------------------
int rcscm_gpu_sphere(rcscm_gpu_ctx* c, int64_t I, int64_t J, int M, const double* X, double* Q, double* Xw) {
  return guarded([&] {
    if (!c) fail(RCSCM_INVALID_INPUT, "ctx must not be NULL");
    if (I < 0 || J < 0 || M < 1) fail(RCSCM_INVALID_INPUT, "sphere: bad shape");
    check_mics(M);
    if (J <= M) fail(RCSCM_INVALID_INPUT, "sphere: need more frames than channels");
    if (I == 0) return;
    const size_t S = static_cast<size_t>(I * J);
    double2* dX = c->X.get<double2>(S * M);
    h2d(c, dX, X, S * M * sizeof(double2));
    double2* dQ = c->il_W.get<double2>(static_cast<size_t>(I) * M * M);
    double2* dXw = c->il_X.get<double2>(S * M);
    c->launched(launch_sphere(c->stream, M, dX, I, J, dQ, dXw));
    if (Q) d2h(c, Q, dQ, static_cast<size_t>(I) * M * M * sizeof(double2));
    if (Xw) d2h(c, Xw, dXw, S * M * sizeof(double2));
    sync(c);
  });
}

// run_ilrma on the device-resident (whitened) dX; results stay in c->il_* (W, A, T, V)
static IlrmaArgs ilrma_dev(rcscm_gpu_ctx* c, const double2* dX, int64_t I, int64_t J, int M, int K, int iters,
                           uint64_t seed) {
  if (K < 1) fail(RCSCM_INVALID_INPUT, "run_ilrma: K must be >= 1");
  if (iters < 0) fail(RCSCM_INVALID_INPUT, "run_ilrma: iters must be >= 0");
  check_mics(M);
  if (K > 16) fail(RCSCM_UNSUPPORTED, "run_ilrma: K > 16 NMF bases is not supported on the GPU");
  const size_t S = static_cast<size_t>(I * J);
  // NMF initialisation exactly as the reference (ilrma.hpp:162-173): one
  // mt19937_64 stream, per source T row-major over (i, k) then V over (k, t)
  std::vector<double> hT(static_cast<size_t>(M) * I * K), hV(static_cast<size_t>(M) * K * J);
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unif(0.1, 1.0);
  for (int n = 0; n < M; ++n) {
    double* Tn = hT.data() + static_cast<size_t>(n) * I * K;
    double* Vn = hV.data() + static_cast<size_t>(n) * K * J;
    for (int64_t i = 0; i < I; ++i)
      for (int k = 0; k < K; ++k) Tn[i + k * I] = unif(rng);
    for (int k = 0; k < K; ++k)
      for (int64_t t = 0; t < J; ++t) Vn[k + t * K] = unif(rng);
  }
  std::vector<double> eye(static_cast<size_t>(I) * M * M * 2, 0.0);
  for (int64_t i = 0; i < I; ++i)
    for (int r = 0; r < M; ++r) eye[2 * (i * M * M + r + r * M)] = 1.0;
  IlrmaArgs a{};
  a.I = I;
  a.J = J;
  a.K = K;
  a.X = dX;
  a.W = c->il_W.get<double2>(static_cast<size_t>(I) * M * M);
  a.A = c->il_A.get<double2>(static_cast<size_t>(I) * M * M);
  a.T = c->il_T.get<double>(hT.size());
  a.V = c->il_V.get<double>(hV.size());
  a.P = c->il_P.get<double>(S * M);
  a.partial = c->il_part.get<double>(static_cast<size_t>(ilrma_partials(I, J)) * M);
  a.mu = c->il_mu.get<double>(M);
  a.Pt = c->il_Pt.get<double>(S * M);
  a.ucov = c->il_ucov.get<double2>(static_cast<size_t>(I) * M * M * M);
  a.err = c->err.get<unsigned long long>(1);
  if (I == 0) return a;
  h2d(c, a.W, eye.data(), eye.size() * sizeof(double));
  h2d(c, a.T, hT.data(), hT.size() * sizeof(double));
  h2d(c, a.V, hV.data(), hV.size() * sizeof(double));
  reset_err(c);
  auto sweeps = [&] {
    c->launched(launch_ilrma_powers(c->stream, a, M));
    for (int pass = 0; pass < 30; ++pass) c->launched(launch_ilrma_nmf(c->stream, a, M), 2);
    for (int it = 0; it < iters; ++it) {
      c->launched(launch_ilrma_nmf(c->stream, a, M), 2);
      c->launched(launch_ilrma_ip_scale(c->stream, a, M), 5);
    }
    c->launched(launch_ilrma_inverse(c->stream, a, M));
  };
  const char* e = std::getenv("RCSCM_ILRMA_GRAPH");
  if (c->stream == nullptr || (e && std::atoi(e) == 0)) {
    sweeps();  // the legacy default stream cannot be captured
  } else {
    ilrma_graph_launch(c, a, M, iters, sweeps);
  }
  check_err(c, J > 0 ? J : 1);
  return a;
}

int rcscm_gpu_run_ilrma(rcscm_gpu_ctx* c, int64_t I, int64_t J, int M, int K, int iters, uint64_t seed,
                        const double* X, double* W, double* A, double* T, double* V) {
  return guarded([&] {
    if (!c) fail(RCSCM_INVALID_INPUT, "ctx must not be NULL");
    if (K < 1) fail(RCSCM_INVALID_INPUT, "run_ilrma: K must be >= 1");
    if (iters < 0) fail(RCSCM_INVALID_INPUT, "run_ilrma: iters must be >= 0");
    if (I < 0 || J < 0 || M < 1) fail(RCSCM_INVALID_INPUT, "run_ilrma: bad shape");
    const size_t S = static_cast<size_t>(I * J);
    double2* dX = c->il_X.get<double2>(S * M);
    if (S) h2d(c, dX, X, S * M * sizeof(double2));
    const IlrmaArgs a = ilrma_dev(c, dX, I, J, M, K, iters, seed);
    if (I == 0) return;
    if (W) d2h(c, W, a.W, static_cast<size_t>(I) * M * M * sizeof(double2));
    if (A) d2h(c, A, a.A, static_cast<size_t>(I) * M * M * sizeof(double2));
    if (T) d2h(c, T, a.T, static_cast<size_t>(M) * I * K * sizeof(double));
    if (V) d2h(c, V, a.V, static_cast<size_t>(M) * K * J * sizeof(double));
    sync(c);
  });
}

// ---- session ------------------------------------------------------------------

// ---- cmd_extract on the device (tools/rcscm.cpp:158-221) ---------------------------
int rcscm_gpu_extract(rcscm_gpu_ctx* c, const rcscm_extract_opts* o, const double* samples, int64_t num_samples,
                      int M, double* target, double* noise, rcscm_extract_result* res) {
  return guarded([&] {
    if (!c || !o || !samples) fail(RCSCM_INVALID_INPUT, "extract: NULL argument");
    if (num_samples <= 0 || M <= 0) fail(RCSCM_INVALID_INPUT, "stft_analyze: empty waveform");
    if (o->iters < 0) fail(RCSCM_INVALID_INPUT, "run_accelerated: iters must be >= 0");
    if (o->backend < 0 || o->backend > 2) fail(RCSCM_INVALID_INPUT, "extract: unknown backend");
    if (o->samples_layout != 0 && o->samples_layout != 1) fail(RCSCM_INVALID_INPUT, "extract: unknown samples_layout");
    check_mics(M);
    const rcscm_hyper h{o->alpha, o->beta};
    // 1. STFT (stft.hpp:50-88)
    const size_t nw = static_cast<size_t>(num_samples) * M;  // samples per waveform
    double* pin = c->ex_pin.get<double>(2 * nw);  // [target | noise] on the way out
    std::memcpy(pin, samples, nw * sizeof(double));
    double* dx = c->st_x.get<double>(nw);
    h2d(c, dx, pin, nw * sizeof(double));
    int win = 0, hop = 0;
    int64_t J = 0, I = 0;
    const bool planar = o->samples_layout == 1;
    stft_analyze_dev(c, dx, num_samples, M, o->sample_rate, o->win_ms, o->hop_ms, &win, &hop, &J, &I, planar);
    const size_t S = static_cast<size_t>(I * J);
    const double2* dX = c->st_X.as<double2>();
    // 2. sphering + ILRMA in the whitened domain (ilrma.hpp:53-73, :145-240)
    if (J <= M) fail(RCSCM_INVALID_INPUT, "sphere: need more frames than channels");
    double2* dQ = c->ex_Q.get<double2>(static_cast<size_t>(I) * M * M);
    double2* dXw = c->il_X.get<double2>(S * M);
    c->launched(launch_sphere(c->stream, M, dX, I, J, dQ, dXw));
    IlrmaArgs a = ilrma_dev(c, dXw, I, J, M, o->nmf_bases, o->ilrma_iters, o->seed);
    // 3. fold the whitening back: W = W_ilrma Q, A = W^{-1} (tools/rcscm.cpp:176-180)
    double2* dW = c->ex_W.get<double2>(static_cast<size_t>(I) * M * M);
    double2* dA = c->ex_A.get<double2>(static_cast<size_t>(I) * M * M);
    c->launched(launch_ilrma_fold(c->stream, a, M, dQ, dW, dA));
    check_err(c, J);
    // 4. target index (model.hpp:43-54) unless given
    int n_h = o->target_index;
    if (n_h >= M) fail(RCSCM_INVALID_INPUT, "extract: target index out of range");
    if (n_h < 0) {
      double* dp = c->ex_pow.get<double>(static_cast<size_t>(M) * I);
      c->launched(launch_target_power(c->stream, M, dX, dW, dA, I, J, dp));
      std::vector<double> pw(static_cast<size_t>(M) * I);
      d2h(c, pw.data(), dp, pw.size() * sizeof(double));
      sync(c);
      double best = -1.0;
      for (int n = 0; n < M; ++n) {
        double p = 0.0;
        for (int64_t i = 0; i < I; ++i) p += pw[n * I + i];
        if (p > best) {
          best = p;
          n_h = n;
        }
      }
    }
    // 5. build_noise_scm + init_params on the device (model.hpp:58-124): the
    //    session's SETUP with T[n_h], V[n_h]
    const int K = o->nmf_bases;
    session_load_impl(c, 1, I, J, M, K, n_h, dX, dW, dA, a.T + static_cast<size_t>(n_h) * I * K,
                      a.V + static_cast<size_t>(n_h) * K * J, cudaMemcpyDeviceToDevice);
    int rc = rcscm_gpu_session_run(c, RCSCM_STAGE_SETUP | RCSCM_STAGE_PRECOMPUTE, 0, &h, o->eps_var);
    if (rc != RCSCM_OK) fail(rc, rcscm_gpu_last_error());
    // 6. the solver (tools/rcscm.cpp:135-142, 184-190)
    std::vector<double> objv;
    const bool want_obj = o->compute_objective != 0;
    // without the early stop the trace stays on the device until the end
    const bool obj_dev = want_obj && !(o->rel_obj_tol > 0.0);
    double* dobj = obj_dev ? c->ex_obj.get<double>(static_cast<size_t>(o->iters) + 1) : nullptr;
    int nobj = 0;
    auto eval = [&] {
      double* slot = obj_dev ? dobj + nobj : nullptr;
      ++nobj;
      return o->backend == 2 ? objective_fast(c, I, J, M, h, slot) : objective(c, I, J, M, h, slot);
    };
    if (want_obj && o->backend == 2) c->launched(launch_logpdet(c->stream, problem(c, 1, I, J, M)));
    if (want_obj) objv.push_back(eval());
    const int step = want_obj ? 1 : o->iters;
    // per-step CUDA events for iter_seconds (solver_accel.hpp:205,227: objective excluded)
    const bool want_secs = res && res->iter_seconds && o->iters > 0;
    struct Events {  // destroyed on every exit path, including fail()
      std::vector<cudaEvent_t> v;
      ~Events() {
        for (cudaEvent_t e : v) cudaEventDestroy(e);
      }
    } evs;
    std::vector<int> ev_n;
    auto event = [&] {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      evs.v.push_back(e);
      CK(cudaEventRecord(e, c->stream));
    };
    int done = 0;
    if (obj_dev && o->backend == 2 && !f32(c) && o->iters > 0) {
      // no early stop: every iteration and its objective in one K2 launch
      if (want_secs) event();
      run_accel_obj(c, I, J, M, o->iters, h, o->eps_var, 0.0, dobj);
      if (want_secs) {
        event();
        ev_n.push_back(o->iters);
      }
      done = o->iters;
      nobj = o->iters + 1;
      objv.resize(nobj);
    }
    while (done < o->iters) {
      const int n = std::min(step, o->iters - done);
      if (want_secs) event();
      if (o->backend == 2) {
        rc = rcscm_gpu_session_run(c, RCSCM_STAGE_ACCEL, n, &h, o->eps_var);
        if (rc != RCSCM_OK) fail(rc, rcscm_gpu_last_error());
        if (f32(c)) params_from_f32(c, S);
      } else if (o->backend == 0) {
        rc = rcscm_gpu_session_run(c, RCSCM_STAGE_NAIVE, n, &h, o->eps_var);
        if (rc != RCSCM_OK) fail(rc, rcscm_gpu_last_error());
      } else {
        c->launched(launch_accel1(c->stream, M, accel1_args(c, I, J, n, h, o->eps_var, 0.0)));
      }
      done += n;
      if (want_secs) {
        event();
        ev_n.push_back(n);
      }
      if (want_obj) {
        objv.push_back(eval());
        const double prev = objv[objv.size() - 2], cur = objv.back();
        if (!obj_dev && std::abs(cur - prev) <= o->rel_obj_tol * std::abs(prev)) break;
      }
    }
    if (obj_dev) d2h(c, objv.data(), dobj, objv.size() * sizeof(double));
    check_err(c, J);
    // 7. Wiener image and noise (wiener.hpp:19-53), then WOLA synthesis of both
    WienerArgs Wa{};
    Wa.nb = I;
    Wa.J = J;
    Wa.X = c->X.as<double2>();
    Wa.a = c->a.as<double2>();
    Wa.b = c->b.as<double2>();
    Wa.Rpp = c->Rpp.as<double2>();
    Wa.r_h = c->rh.as<double>();
    Wa.r_u = c->ru.as<double>();
    Wa.lambda = c->lam.as<double>();
    Wa.dry = c->dry.get<double2>(S);
    Wa.image = c->image.get<double2>(S * M);
    Wa.noise = c->noise.get<double2>(S * M);
    c->launched(launch_wiener(c->stream, M, Wa, true, true));
    // both waveforms synthesised into one device buffer, one D2H into the
    // pinned stage, then host copies into the caller's buffers
    double* dout = c->ex_out.get<double>(2 * nw);
    if (target) stft_synth_dev(c, Wa.image, I, J, M, win, hop, num_samples, dout, planar);
    if (noise) stft_synth_dev(c, Wa.noise, I, J, M, win, hop, num_samples, dout + nw, planar);
    if (target && noise) {
      d2h(c, pin, dout, 2 * nw * sizeof(double));
    } else if (target || noise) {
      d2h(c, target ? pin : pin + nw, target ? dout : dout + nw, nw * sizeof(double));
    }
    sync(c);
    if (target && noise) {
      std::thread th([&] { std::memcpy(noise, pin + nw, nw * sizeof(double)); });
      std::memcpy(target, pin, nw * sizeof(double));
      th.join();
    } else if (target) {
      std::memcpy(target, pin, nw * sizeof(double));
    } else if (noise) {
      std::memcpy(noise, pin + nw, nw * sizeof(double));
    }
    if (res) {
      res->target_index = n_h;
      res->n_iters = done;
      res->bins = I;
      res->frames = J;
      if (res->objective && want_obj)
        std::memcpy(res->objective, objv.data(), objv.size() * sizeof(double));
      res->n_objective = static_cast<int>(objv.size());
      int k = 0;
      for (size_t q = 0; q < ev_n.size(); ++q) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, evs.v[2 * q], evs.v[2 * q + 1]));
        for (int r = 0; r < ev_n[q]; ++r) res->iter_seconds[k++] = 1e-3 * ms / ev_n[q];
      }
    }
  });
}


}  // extern "C"
