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
  std::printf("shim_check: naive r_h %.17g (want %.17g) accel==naive %d wiener %d throws %d\n",
              naive.params.r_h[0], want, ok2, ok3, threw);
  return (ok1 && ok2 && ok3 && threw) ? 0 : 1;
}
