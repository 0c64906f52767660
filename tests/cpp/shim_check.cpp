// shim_check.cpp -- the C++ front end (include/rcscm_gpu.hpp) used the way the
// reference's own call sites use their entry points (tools/rcscm.cpp:135-142,
// cmd_extract :158-221): a tiny scalar instance with the known answer of
// test_solver_naive.cpp:44-58 (r^ = 5/3), then accel == naive and the Wiener
// output. Compiled by __graft_entry__.build(); executed by tests (GPU only).
#include <cmath>
#include <cstdio>

#include "../../include/rcscm_gpu.hpp"

using namespace rcscm::gpu;

int main() {
  Context ctx(0);
  RcscmInputs in;
  in.bins = 1;
  in.mics = 1;
  in.a = {cplx(1.0, 0.0)};
  in.b = {cplx(1.0, 0.0)};
  in.R_prime = {cplx(0.0, 0.0)};
  in.R_prime_pinv = {cplx(0.0, 0.0)};
  RcscmParams p0;
  p0.bins = 1;
  p0.frames = 1;
  p0.r_h = {1.0};
  p0.r_u = {1.0};
  p0.lambda = {2.0};
  Spectrogram X;
  X.bins = 1;
  X.frames = 1;
  X.mics = 1;
  X.data = {cplx(3.0, 0.0)};
  SolverOptions opt;
  opt.iters = 1;
  const SolverResult naive = run_naive(ctx, in, p0, Hyperparams{}, X, opt);
  const SolverResult accel = run_algorithm2(ctx, in, p0, Hyperparams{}, X, opt);
  const double want = (5.0 / 3.0 + 1e-16) / 3.1;
  const bool ok1 = std::abs(naive.params.r_h[0] - want) < 1e-12 * want;
  const bool ok2 = std::abs(accel.params.r_h[0] - naive.params.r_h[0]) < 1e-12 * want &&
                   std::abs(accel.params.r_u[0] - naive.params.r_u[0]) < 1e-12 &&
                   std::abs(accel.params.lambda[0] - naive.params.lambda[0]) < 1e-12;
  const ExtractionResult ex = extract_target(ctx, in, accel.params, X);
  const bool ok3 = std::isfinite(ex.dry[0].real()) && std::abs(ex.image.data[0] - ex.dry[0]) < 1e-15;
  bool threw = false;
  try {
    opt.iters = -1;
    run_algorithm2(ctx, in, p0, Hyperparams{}, X, opt);
  } catch (const InvalidInputError&) {
    threw = true;
  }
  // Algorithm 1 agrees with the naive rule on the scalar case (acceptance.cpp:34-65)
  opt.iters = 1;
  const SolverResult alg1 = run_algorithm1(ctx, in, p0, Hyperparams{}, X, opt);
  const bool ok4 = std::abs(alg1.params.r_h[0] - naive.params.r_h[0]) < 1e-12 * want &&
                   std::abs(alg1.params.lambda[0] - naive.params.lambda[0]) < 1e-12;
  // STFT round trip (test_stft.cpp:82-97): a 440 Hz tone on 2 channels
  Waveform w;
  w.channels = 2;
  w.num_samples = 16000;
  w.samples.resize(2 * 16000);
  for (int64_t t = 0; t < w.num_samples; ++t)
    for (int ch = 0; ch < 2; ++ch) w.samples[ch + 2 * t] = std::sin(2.0 * M_PI * 440.0 * (t + ch) / 16000.0);
  const Spectrogram S = stft_analyze(ctx, w, 64.0, 32.0);
  const Waveform r = stft_synthesize(ctx, S, 64.0, 32.0);
  double err = 0.0, ref = 0.0;
  for (int64_t k = 2 * 1024; k < 2 * (16000 - 1024); ++k) {
    err += (r.samples[k] - w.samples[k]) * (r.samples[k] - w.samples[k]);
    ref += w.samples[k] * w.samples[k];
  }
  const bool ok5 = S.bins == 513 && S.frames == 33 && r.num_samples == w.num_samples && std::sqrt(err / ref) < 1e-8;
  // a device list (here device 0 twice): bins sharded over two contexts, the
  // result bitwise equal to one device -- 3 bins of the scalar case
  Context multi(std::vector<int>{0, 0});
  RcscmInputs in3 = in;
  in3.bins = 3;
  in3.a.assign(3, cplx(1.0, 0.0));
  in3.b.assign(3, cplx(1.0, 0.0));
  in3.R_prime.assign(3, cplx(0.0, 0.0));
  in3.R_prime_pinv.assign(3, cplx(0.0, 0.0));
  RcscmParams q0 = p0;
  q0.bins = 3;
  q0.r_h = {1.0, 2.0, 0.5};
  q0.r_u = {1.0, 0.7, 1.5};
  q0.lambda = {2.0, 1.0, 3.0};
  Spectrogram X3 = X;
  X3.bins = 3;
  X3.data = {cplx(3.0, 0.0), cplx(1.0, -2.0), cplx(0.5, 0.25)};
  opt.iters = 4;
  const SolverResult one = run_algorithm2(ctx, in3, q0, Hyperparams{}, X3, opt);
  const SolverResult two = run_algorithm2(multi, in3, q0, Hyperparams{}, X3, opt);
  const bool ok6 = one.params.r_h == two.params.r_h && one.params.r_u == two.params.r_u &&
                   one.params.lambda == two.params.lambda;
  std::printf("shim_check: naive r_h %.17g (want %.17g) accel==naive %d wiener %d throws %d alg1 %d stft %d "
              "devices %d\n",
              naive.params.r_h[0], want, ok2, ok3, threw, ok4, ok5, ok6);
  return (ok1 && ok2 && ok3 && threw && ok4 && ok5 && ok6) ? 0 : 1;
}
