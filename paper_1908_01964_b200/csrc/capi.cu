// capi.cu -- host side of the rcscm B200 path: the C ABI of include/rcscm_gpu.h.
//
// Each reference entry point (model.hpp, solver_naive.hpp, solver_accel.hpp,
// wiener.hpp) becomes: host->device copies of the caller's reference-layout
// buffers, one transpose of the I x J column-major parameters into the
// device's bin-major layout, the CUDA kernels, and the way back. There is no
// CPU fallback: every numeric step runs in the kernels launched through
// launch.h (setup_launch.cu, accel_launch.cu, naive_launch.cu, stream_launch.cu).
#include <chrono>
#include <cstdio>
#include <thread>

#include "capi_internal.h"

using namespace rcscm_capi;

namespace rcscm_capi {

thread_local std::string g_last_error;

void h2d(rcscm_gpu_ctx* c, void* dst, const void* src, size_t bytes) {
  if (bytes) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
}
void d2h(rcscm_gpu_ctx* c, void* dst, const void* src, size_t bytes) {
  if (bytes && dst) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
}
void d2d(rcscm_gpu_ctx* c, void* dst, const void* src, size_t bytes) {
  if (bytes) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, c->stream));
}
void sync(rcscm_gpu_ctx* c) { CK(cudaStreamSynchronize(c->stream)); }
void h2d_ij(rcscm_gpu_ctx* c, void* dst, const void* src, int64_t I, int64_t J, size_t esz) {
  const int64_t ld = c->ldh > I ? c->ldh : I;
  if (ld == I) return h2d(c, dst, src, static_cast<size_t>(I * J) * esz);
  if (I * J) CK(cudaMemcpy2DAsync(dst, I * esz, src, ld * esz, I * esz, J, cudaMemcpyHostToDevice, c->stream));
}
void d2h_ij(rcscm_gpu_ctx* c, void* dst, const void* src, int64_t I, int64_t J, size_t esz) {
  const int64_t ld = c->ldh > I ? c->ldh : I;
  if (ld == I) return d2h(c, dst, src, static_cast<size_t>(I * J) * esz);
  if (I * J && dst) CK(cudaMemcpy2DAsync(dst, ld * esz, src, I * esz, I * esz, J, cudaMemcpyDeviceToHost, c->stream));
}

void reset_err(rcscm_gpu_ctx* c) {
  unsigned long long* e = c->err.get<unsigned long long>(1);
  CK(cudaMemsetAsync(e, 0xFF, sizeof(unsigned long long), c->stream));
}

// Decode the device error word (after a sync) into the reference's messages.
int decode_err(unsigned long long key, int64_t J, std::string* msg) {
  if (key == ~0ull) return RCSCM_OK;
  const unsigned code = static_cast<unsigned>(key & 0xF);
  const unsigned aux = static_cast<unsigned>((key >> 4) & 0xF);
  const long long slot = static_cast<long long>(key >> 8);
  const long long bin = J > 0 ? slot / J : slot, t = J > 0 ? slot % J : 0;
  const std::string bs = std::to_string(bin), ts = std::to_string(t);
  switch (code) {
    case kErrEStepSingular:
      *msg = "e_step: singular covariance at bin " + bs + ", frame " + ts;
      return RCSCM_NUMERICAL;
    case kErrMStepSingular:
      *msg = "m_step: singular R^(u) at bin " + bs;
      return RCSCM_NUMERICAL;
    case kErrNullVector:
      *msg = "build_noise_scm: frequency bin " + bs +
             ": null_eigenvector: expected exactly one near-zero eigenvalue, found " + std::to_string(aux);
      return RCSCM_INVALID_INPUT;
    case kErrNotPsd:
      *msg = "build_noise_scm: frequency bin " + bs + ": pseudo_inverse_psd: matrix is not PSD";
      return RCSCM_INVALID_INPUT;
    case kErrObjectiveNotPd:
      *msg = "map_objective: R^(x) not PD at bin " + bs + ", frame " + ts;
      return RCSCM_NUMERICAL;
    case kErrObjectiveNonFinite:
      *msg = "map_objective: non-finite at bin " + bs + ", frame " + ts;
      return RCSCM_NUMERICAL;
    case kErrEigNoConverge:
      *msg = "hermitian_eig: eigensolver failed to converge (bin " + bs + ")";
      return RCSCM_NUMERICAL;
    case kErrFirstStageLambda:
      *msg = "rho_first_stage: nonpositive lambda at bin " + bs;
      return RCSCM_NUMERICAL;
    case kErrFirstStageSingular:
      *msg = "rho_first_stage: singular R^(u) at bin " + bs;
      return RCSCM_NUMERICAL;
    case kErrIlrmaSpatial:
      *msg = "run_ilrma: singular spatial update at frequency bin " + bs;
      return RCSCM_NUMERICAL;
    case kErrIlrmaDemix:
      *msg = "run_ilrma: singular demixing matrix at frequency bin " + bs;
      return RCSCM_NUMERICAL;
    default:
      *msg = "device error code " + std::to_string(code);
      return RCSCM_NUMERICAL;
  }
}

void check_err(rcscm_gpu_ctx* c, int64_t J) {
  // into a page-locked word: a direct DMA instead of the driver's pageable staging
  unsigned long long* hk = c->err_pin.get<unsigned long long>(1);
  *hk = ~0ull;
  CK(cudaMemcpyAsync(hk, c->err.as<unsigned long long>(), sizeof(*hk), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  unsigned long long key = *hk;
  if (key != ~0ull && c->bin_offset && J > 0)  // a bin range of a sharded call: global slot
    key = (((key >> 8) + static_cast<unsigned long long>(c->bin_offset * J)) << 8) | (key & 0xFFull);
  std::string msg;
  const int rc = decode_err(key, J, &msg);
  if (rc != RCSCM_OK) fail(rc, msg);
}

DevProblem problem(rcscm_gpu_ctx* c, int64_t B, int64_t I, int64_t J, int M) {
  DevProblem P{};
  P.nb = B * I;
  P.I = I;
  P.J = J;
  P.M = M;
  P.K = c->sK;
  P.n_h = c->sn_h;
  P.X = c->X.as<double2>();
  P.W = c->W.as<double2>();
  P.A = c->A.as<double2>();
  P.T = c->T.as<double>();
  P.V = c->V.as<double>();
  P.a = c->a.as<double2>();
  P.b = c->b.as<double2>();
  P.Rp = c->Rp.as<double2>();
  P.Rpp = c->Rpp.as<double2>();
  P.power = c->power.as<double>();
  P.sigma_ab = c->sab.as<double2>();
  P.tau_aa = c->taa.as<double>();
  P.sigma_bx = c->sbx.as<double2>();
  P.tau_ax = c->tax.as<double2>();
  P.tau_xx = c->txx.as<double>();
  P.r_h = c->rh.as<double>();
  P.r_u = c->ru.as<double>();
  P.lambda = c->lam.as<double>();
  P.logpdet = c->lpd.as<double>();
  P.err = c->err.as<unsigned long long>();
  return P;
}

// Allocate every per-bin / per-slot device buffer for nb bins x J frames.
void alloc_problem(rcscm_gpu_ctx* c, int64_t nb, int64_t J, int M) {
  const size_t S = static_cast<size_t>(nb * J);
  c->X.get<double2>(S * M);
  c->a.get<double2>(nb * M);
  c->b.get<double2>(nb * M);
  c->Rp.get<double2>(nb * M * M);
  c->Rpp.get<double2>(nb * M * M);
  c->power.get<double>(nb * M);
  c->sab.get<double2>(nb);
  c->taa.get<double>(nb);
  c->sbx.get<double2>(S);
  c->tax.get<double2>(S);
  c->txx.get<double>(S);
  c->rh.get<double>(S);
  c->ru.get<double>(S);
  c->lam.get<double>(nb);
  c->lpd.get<double>(nb);
  c->err.get<unsigned long long>(1);
}

bool f32(const rcscm_gpu_ctx* c) { return c->precision == RCSCM_C64; }

// complex64 mode: single-precision copies of x and of the parameters
void alloc_f32(rcscm_gpu_ctx* c, int64_t nb, int64_t J, int M) {
  const size_t S = static_cast<size_t>(nb * J);
  c->Xf.get<float2>(S * M);
  c->sbxf.get<float2>(S);
  c->taxf.get<float2>(S);
  c->txxf.get<float>(S);
  c->rhf.get<float>(S);
  c->ruf.get<float>(S);
}
void x_to_f32(rcscm_gpu_ctx* c, size_t S, int M) {
  c->launched(launch_d2f(c->stream, c->X.as<double>(), c->Xf.as<float>(), static_cast<int64_t>(2 * S * M)));
}
void params_to_f32(rcscm_gpu_ctx* c, size_t S, const double* rh, const double* ru) {
  c->launched(launch_d2f(c->stream, rh, c->rhf.as<float>(), static_cast<int64_t>(S)));
  c->launched(launch_d2f(c->stream, ru, c->ruf.as<float>(), static_cast<int64_t>(S)));
}
void params_from_f32(rcscm_gpu_ctx* c, size_t S) {
  c->launched(launch_f2d(c->stream, c->rhf.as<float>(), c->rh.as<double>(), static_cast<int64_t>(S)));
  c->launched(launch_f2d(c->stream, c->ruf.as<float>(), c->ru.as<double>(), static_cast<int64_t>(S)));
}
// sigma / tau precompute in the context's precision
void precompute(rcscm_gpu_ctx* c, const DevProblem& P, double eps) {
  if (f32(c))
    c->launched(launch_slots_pre_f32(c->stream, P, c->Xf.as<float2>(), c->sbxf.as<float2>(), c->taxf.as<float2>(),
                                     c->txxf.as<float>()));
  else
    c->launched(launch_slots(c->stream, P, false, true, eps));
}

AccelArgs accel_args(rcscm_gpu_ctx* c, int64_t nb, int64_t J, int M, int iters, const rcscm_hyper& h, double eps,
                     double gamma_fault) {
  AccelArgs A{};
  A.nb = nb;
  A.J = J;
  A.iters = iters;
  A.inv_M = 1.0 / static_cast<double>(M);
  A.k1 = 1.0 / (h.alpha + 2.0);
  A.k2 = h.beta / (h.alpha + 2.0);
  A.eps = eps;
  A.gamma_fault = gamma_fault;
  A.sigma_ab = c->sab.as<double2>();
  A.tau_aa = c->taa.as<double>();
  A.sigma_bx = c->sbx.as<double2>();
  A.tau_ax = c->tax.as<double2>();
  A.tau_xx = c->txx.as<double>();
  A.r_h = c->rh.as<double>();
  A.r_u = c->ru.as<double>();
  A.lambda = c->lam.as<double>();
  A.sigma_bx_f = c->sbxf.as<float2>();
  A.tau_ax_f = c->taxf.as<float2>();
  A.tau_xx_f = c->txxf.as<float>();
  A.r_h_f = c->rhf.as<float>();
  A.r_u_f = c->ruf.as<float>();
  A.r_h_in = A.r_h;
  A.r_u_in = A.r_u;
  A.lambda_in = A.lambda;
  A.r_h_f_in = A.r_h_f;
  A.r_u_f_in = A.r_u_f;
  return A;
}

// K2 reads x and forms sigma / tau itself (fused precompute) for the bins
// [b0, b0 + A.nb) of the context's arrays; keep_forms also stores the forms
// (and sigma_ab, tau_aa) for later stages.
void set_fused(rcscm_gpu_ctx* c, AccelArgs& A, int64_t b0, int64_t J, int M, bool keep_forms) {
  const size_t off = static_cast<size_t>(b0 * J);
  A.X = c->X.as<double2>() + off * M;
  A.a_in = c->a.as<double2>() + b0 * M;
  A.b_in = c->b.as<double2>() + b0 * M;
  A.Rpp_in = c->Rpp.as<double2>() + b0 * M * M;
  if (keep_forms) {
    A.sigma_ab_w = c->sab.as<double2>() + b0;
    A.tau_aa_w = c->taa.as<double>() + b0;
    A.sigma_bx_w = c->sbx.as<double2>() + off;
    A.tau_ax_w = c->tax.as<double2>() + off;
    A.tau_xx_w = c->txx.as<double>() + off;
  }
}

void run_accel(rcscm_gpu_ctx* c, const AccelArgs& A, int prem = 0) {
  if (A.nb * A.J == 0) return;
  AccelCfg g = choose_accel_cfg(A.J, f32(c));
  g.prem = prem;
  accel_one_warp(g, A.nb);
  if (!g.cl) {
    // longer than a 16-CTA cluster holds (32768 frames): stream the iterate
    // through HBM (two launches per iteration; complex128, sigma / tau from K1)
    if (f32(c) || prem)
      fail(RCSCM_UNSUPPORTED, "frames = " + std::to_string(A.J) +
                                  " exceeds the on-chip accel kernel capacity (16 x 2048) in this mode");
    if (A.ld_p) fail(RCSCM_UNSUPPORTED, "streaming accel kernel: column-major parameters");
    double* part = c->st_part.get<double>(static_cast<size_t>(A.nb * accel_stream_chunks(A.J)));
    double* lam = c->st_lam.get<double>(static_cast<size_t>(4 * A.nb));
    int n = 0;
    const cudaError_t e = launch_accel_stream(c->stream, A, part, lam, &n);
    c->launched(e, n);
    return;
  }
  c->launched(launch_accel(c->stream, A, g));
}

Accel1Args accel1_args(rcscm_gpu_ctx* c, int64_t nb, int64_t J, int iters, const rcscm_hyper& h, double eps,
                       double gamma_fault) {
  Accel1Args A{};
  A.nb = nb;
  A.J = J;
  A.iters = iters;
  A.alpha2 = h.alpha + 2.0;
  A.beta = h.beta;
  A.eps = eps;
  A.gamma_fault = gamma_fault;
  A.X = c->X.as<double2>();
  A.a = c->a.as<double2>();
  A.b = c->b.as<double2>();
  A.Rp = c->Rp.as<double2>();
  A.r_h = c->rh.as<double>();
  A.r_u = c->ru.as<double>();
  A.lambda = c->lam.as<double>();
  const size_t S = static_cast<size_t>(nb * J);
  A.rho_ax = c->scratch.get<double2>(S);
  A.sigma_bx = c->sbx.get<double2>(S);
  A.gamma = c->gam.get<double>(S);
  A.err = c->err.as<unsigned long long>();
  return A;
}

NaiveArgs naive_args(rcscm_gpu_ctx* c, int64_t nb, int64_t J, int iters, const rcscm_hyper& h, double eps) {
  NaiveArgs N{};
  N.nb = nb;
  N.J = J;
  N.iters = iters;
  N.alpha = h.alpha;
  N.beta = h.beta;
  N.eps = eps;
  N.X = c->X.as<double2>();
  N.a = c->a.as<double2>();
  N.b = c->b.as<double2>();
  N.Rp = c->Rp.as<double2>();
  N.r_h = c->rh.as<double>();
  N.r_u = c->ru.as<double>();
  N.lambda = c->lam.as<double>();
  N.scratch = c->scratch.get<double2>(static_cast<size_t>(nb * J));
  N.err = c->err.as<unsigned long long>();
  return N;
}

// Objective of the current device state -> host double (synchronizes).
double objective(rcscm_gpu_ctx* c, int64_t nb, int64_t J, int M, const rcscm_hyper& h, double* dev_out) {
  if (nb * J == 0) return 0.0;
  ObjArgs O{};
  O.nb = nb;
  O.J = J;
  O.alpha = h.alpha;
  O.beta = h.beta;
  O.X = c->X.as<double2>();
  O.a = c->a.as<double2>();
  O.b = c->b.as<double2>();
  O.Rp = c->Rp.as<double2>();
  O.r_h = c->rh.as<double>();
  O.r_u = c->ru.as<double>();
  O.lambda = c->lam.as<double>();
  O.partial = c->partial.get<double>(static_cast<size_t>(nb * ((J + 127) / 128)));
  O.err = c->err.as<unsigned long long>();
  int64_t np = 0;
  c->launched(launch_objective(c->stream, M, O, &np));
  double* out = dev_out ? dev_out : c->obj.get<double>(1);
  c->launched(launch_sum_partials(c->stream, O.partial, np, out));
  if (dev_out) return 0.0;
  double v = 0.0;
  d2h(c, &v, out, sizeof(double));
  check_err(c, J);
  return v;
}

// O(1)-per-slot objective from the resident sigma/tau precompute (needs
// logpdet, see launch_logpdet); synchronizes.
double objective_fast(rcscm_gpu_ctx* c, int64_t nb, int64_t J, int M, const rcscm_hyper& h, double* dev_out) {
  if (nb * J == 0) return 0.0;
  ObjFastArgs O{};
  O.nb = nb;
  O.J = J;
  O.M = M;
  O.alpha = h.alpha;
  O.beta = h.beta;
  O.sigma_ab = c->sab.as<double2>();
  O.tau_aa = c->taa.as<double>();
  O.sigma_bx = c->sbx.as<double2>();
  O.tau_ax = c->tax.as<double2>();
  O.tau_xx = c->txx.as<double>();
  O.logpdet = c->lpd.as<double>();
  O.r_h = c->rh.as<double>();
  O.r_u = c->ru.as<double>();
  O.lambda = c->lam.as<double>();
  O.partial = c->partial.get<double>(static_cast<size_t>(nb * ((J + 127) / 128)));
  O.err = c->err.as<unsigned long long>();
  int64_t np = 0;
  c->launched(launch_objective_fast(c->stream, O, &np));
  double* out = dev_out ? dev_out : c->obj.get<double>(1);
  c->launched(launch_sum_partials(c->stream, O.partial, np, out));
  if (dev_out) return 0.0;
  double v = 0.0;
  d2h(c, &v, out, sizeof(double));
  check_err(c, J);
  return v;
}

void run_accel_obj(rcscm_gpu_ctx* c, int64_t I, int64_t J, int M, int iters, const rcscm_hyper& h, double eps,
                   double gamma_fault, double* dobj, double* trh, double* tru, double* trl) {
  if (iters <= 0 || I * J == 0) return;
  AccelArgs A = accel_args(c, I, J, M, iters, h, eps, gamma_fault);
  const AccelCfg g = choose_accel_cfg(J, false);
  if (!g.cl)
    fail(RCSCM_UNSUPPORTED, "frames = " + std::to_string(J) + " exceeds the on-chip accel kernel capacity (16 x 2048)");
  const int64_t nparts = I * g.cl;  // one partial per CTA and iteration
  A.obj_part = c->obj_part.get<double>(static_cast<size_t>(iters) * nparts);
  A.logpdet = c->lpd.as<double>();
  A.alpha = h.alpha;
  A.beta = h.beta;
  A.mics = M;
  A.err = c->err.as<unsigned long long>();
  A.traj_r_h = trh;
  A.traj_r_u = tru;
  A.traj_lambda = trl;
  c->launched(launch_accel(c->stream, A, g));
  c->launched(launch_sum_rows(c->stream, A.obj_part, iters, nparts, dobj + 1));
}

// ---- argument validation ---------------------------------------------------------
void validate_inputs(const rcscm_inputs* in, bool need_rp, bool need_rpp) {
  if (!in) fail(RCSCM_INVALID_INPUT, "inputs must not be NULL");
  if (in->num_bins < 0 || in->frames < 0) fail(RCSCM_INVALID_INPUT, "negative shape");
  if (in->mics < 1) fail(RCSCM_INVALID_INPUT, "mics must be >= 1");
  if (in->num_bins > 0 && in->frames < 1) fail(RCSCM_INVALID_INPUT, "frames must be >= 1");
  if (in->num_bins > 0) {
    if (!in->a || !in->b) fail(RCSCM_INVALID_INPUT, "inputs.a / inputs.b must not be NULL");
    if (need_rp && !in->R_prime) fail(RCSCM_INVALID_INPUT, "inputs.R_prime must not be NULL");
    if (need_rpp && !in->R_prime_pinv) fail(RCSCM_INVALID_INPUT, "inputs.R_prime_pinv must not be NULL");
  }
  check_mics(in->mics);
}

// Upload inputs + params0 into the context's device buffers (device layout).
void upload_model(rcscm_gpu_ctx* c, const rcscm_inputs* in, const rcscm_params* p, const double* X, bool rp,
                  bool rpp) {
  const int64_t I = in->num_bins, J = in->frames;
  const int M = in->mics;
  alloc_problem(c, I, J, M);
  const size_t S = static_cast<size_t>(I * J);
  h2d(c, c->X.p, X, S * M * sizeof(double2));
  h2d(c, c->a.p, in->a, I * M * sizeof(double2));
  h2d(c, c->b.p, in->b, I * M * sizeof(double2));
  if (rp) h2d(c, c->Rp.p, in->R_prime, I * M * M * sizeof(double2));
  if (rpp) h2d(c, c->Rpp.p, in->R_prime_pinv, I * M * M * sizeof(double2));
  if (p) {
    double* t1 = c->tmp.get<double>(S);
    double* t2 = c->tmp2.get<double>(S);
    h2d_ij(c, t1, p->r_h, I, J, sizeof(double));
    h2d_ij(c, t2, p->r_u, I, J, sizeof(double));
    c->launched(launch_to_bt(c->stream, t1, c->rh.as<double>(), 1, I, J));
    c->launched(launch_to_bt(c->stream, t2, c->ru.as<double>(), 1, I, J));
    h2d(c, c->lam.p, p->lambda, I * sizeof(double));
  }
}

void download_params(rcscm_gpu_ctx* c, int64_t I, int64_t J, rcscm_params* out) {
  const size_t S = static_cast<size_t>(I * J);
  double* t1 = c->tmp.get<double>(S);
  double* t2 = c->tmp2.get<double>(S);
  c->launched(launch_to_ij(c->stream, c->rh.as<double>(), t1, 1, I, J));
  c->launched(launch_to_ij(c->stream, c->ru.as<double>(), t2, 1, I, J));
  d2h_ij(c, out->r_h, t1, I, J, sizeof(double));
  d2h_ij(c, out->r_u, t2, I, J, sizeof(double));
  d2h(c, out->lambda, c->lam.p, I * sizeof(double));
}

void validate_opts(const rcscm_solver_opts* opt, const char* who) {
  if (!opt) fail(RCSCM_INVALID_INPUT, std::string(who) + ": options must not be NULL");
  if (opt->iters < 0) fail(RCSCM_INVALID_INPUT, std::string(who) + ": iters must be >= 0");
}

// Copy/compute-overlapped run_algorithm2 (no objective, no trajectory). A copy
// stream uploads the small per-bin inputs and the whole r_h / r_u / lambda
// (contiguous), then x chunk by chunk of bins; the compute stream waits for each
// x chunk and runs K2 with the sigma / tau precompute fused and r_h / r_u read
// and written in place in the caller's I x J column-major layout (other K2
// variants: transpose -> sigma/tau -> K2 -> transpose back) on that chunk while
// the next chunk is still in flight; each chunk's results go back as 2D row
// blocks on a D2H stream. Chunks own disjoint bin ranges of every buffer and
// the per-bin arithmetic is unchanged, so the result is bitwise identical to
// the single-shot path. Returns false when the problem is too small to split.
bool run_accel_pipelined(rcscm_gpu_ctx* c, const rcscm_inputs* in, const rcscm_params* p0,
                         const rcscm_hyper* hyper, const double* X, const rcscm_solver_opts* opt,
                         rcscm_params* out, std::vector<double>* secs) {
  const int64_t I = in->num_bins, J = in->frames;
  const int M = in->mics;
  const char* e_ch = std::getenv("RCSCM_PIPELINE_CHUNKS");
  int nch = e_ch ? std::atoi(e_ch) : static_cast<int>(std::min<int64_t>(8, I / 128));
  nch = static_cast<int>(std::min<int64_t>(std::min(nch, kMaxChunks), I));  // no empty chunks
  if (nch < 2) return false;
  AccelCfg g = choose_accel_cfg(J);
  if (!g.cl) return false;
  if (accel_fusable(g, M) && opt->iters > 0) g.prem = M;  // one kernel per chunk: precompute fused into K2
  accel_one_warp(g, I / nch);
  for (int k = 0; k < 4; ++k)
    if (!c->aux[k]) CK(cudaStreamCreateWithFlags(&c->aux[k], cudaStreamNonBlocking));
  for (int k = 0; k < kMaxChunks + 6; ++k)
    if (!c->evx[k]) CK(cudaEventCreateWithFlags(&c->evx[k], cudaEventDisableTiming));
  for (int k = 0; k < 2 * kMaxChunks; ++k)
    if (!c->evt[k]) CK(cudaEventCreate(&c->evt[k]));
  // H2D alternates between two copy streams (two DMA engines run concurrently;
  // one alone reaches about half of the PCIe rate); K2 runs on cs per chunk
  cudaStream_t cpy[2] = {c->aux[0], c->aux[2]}, cs = c->aux[1];
  alloc_problem(c, I, J, M);
  const size_t S = static_cast<size_t>(I * J);
  double* t1 = c->tmp.get<double>(S);
  double* t2 = c->tmp2.get<double>(S);
  const auto th0 = std::chrono::steady_clock::now();  // RCSCM_DEBUG_TIMING: host enqueue time
  reset_err(c);
  CK(cudaEventRecord(c->ev0, c->stream));
  CK(cudaEventRecord(c->evx[0], c->stream));
  for (cudaStream_t q : {cpy[0], cpy[1], cs}) CK(cudaStreamWaitEvent(q, c->evx[0], 0));
  auto up = [&](int e, void* dst, const void* src, size_t bytes) {
    if (bytes) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, cpy[e]));
  };
  const int64_t ldh = c->ldh > I ? c->ldh : I;  // host leading dimension of r_h / r_u
  auto up_ij = [&](int e, double* dst, const double* src) {
    if (ldh == I) return up(e, dst, src, S * sizeof(double));
    CK(cudaMemcpy2DAsync(dst, I * sizeof(double), src, ldh * sizeof(double), I * sizeof(double), J,
                         cudaMemcpyHostToDevice, cpy[e]));
  };
  // r_h0 / r_u0 (I x J col-major: every chunk needs all of both) first, one per engine
  up_ij(0, t1, p0->r_h);
  up_ij(1, t2, p0->r_u);
  up(0, c->lam.p, p0->lambda, I * sizeof(double));
  up(0, c->a.p, in->a, I * M * sizeof(double2));
  up(1, c->b.p, in->b, I * M * sizeof(double2));
  up(1, c->Rpp.p, in->R_prime_pinv, I * M * M * sizeof(double2));
  CK(cudaEventRecord(c->evx[1], cpy[0]));
  CK(cudaEventRecord(c->evx[kMaxChunks + 3], cpy[1]));
  for (int ch = 0; ch < nch; ++ch) {
    const int64_t i0 = I * ch / nch, i1 = I * (ch + 1) / nch;
    up(ch & 1, c->X.as<double2>() + i0 * J * M, X + 2 * i0 * J * M, (i1 - i0) * J * M * sizeof(double2));
    CK(cudaEventRecord(c->evx[3 + ch], cpy[ch & 1]));
  }
  const DevProblem full = problem(c, 1, I, J, M);
  const AccelArgs afull = accel_args(c, I, J, M, opt->iters, *hyper, opt->eps_var, opt->gamma_fault);
  CK(cudaStreamWaitEvent(cs, c->evx[1], 0));
  CK(cudaStreamWaitEvent(cs, c->evx[kMaxChunks + 3], 0));
  // output segments (RCSCM_D2H_SEGS; default one per chunk, measured fastest on
  // config 1: 1.41 -> 1.25 ms per call): groups of consecutive chunks
  const char* e_sg = std::getenv("RCSCM_D2H_SEGS");
  const int nseg = std::max(1, std::min(nch, e_sg ? std::atoi(e_sg) : nch));
  auto seg_of = [&](int ch) { return ch * nseg / nch; };
  auto seg_first = [&](int sg) {  // first chunk of segment sg
    int ch = 0;
    while (seg_of(ch) < sg) ++ch;
    return ch;
  };
  cudaStream_t cd = c->aux[3];
  CK(cudaStreamWaitEvent(cd, c->evx[0], 0));
  int64_t d_done = 0;  // bins already sent back
  auto send_rows = [&](cudaStream_t q, int64_t b0, int64_t b1) {  // bins [b0, b1) of r_h / r_u to the caller
    if (b1 <= b0) return;
    for (auto pr : {std::make_pair(out->r_h, t1), std::make_pair(out->r_u, t2)})
      CK(cudaMemcpy2DAsync(pr.first + b0, ldh * sizeof(double), pr.second + b0, I * sizeof(double),
                           (b1 - b0) * sizeof(double), J, cudaMemcpyDeviceToHost, q));
  };
  for (int ch = 0; ch < nch; ++ch) {
    const int64_t i0 = I * ch / nch, i1 = I * (ch + 1) / nch, Ic = i1 - i0;
    if (Ic == 0) continue;
    const size_t off = static_cast<size_t>(i0 * J);
    CK(cudaStreamWaitEvent(cs, c->evx[3 + ch], 0));
    // the fused K2 reads and writes r_h / r_u in the caller's I x J column-major
    // layout (ld_p = I) in place in t1 / t2; other variants go through the
    // bin-major arrays with transposes around them
    const bool colmajor = g.prem != 0;
    if (!colmajor) {
      c->launched(launch_to_bt(cs, t1 + i0, c->rh.as<double>() + off, 1, Ic, J, I));
      c->launched(launch_to_bt(cs, t2 + i0, c->ru.as<double>() + off, 1, Ic, J, I));
    }
    DevProblem P = full;
    P.nb = Ic;
    P.I = Ic;
    P.X += off * M;
    P.a += i0 * M;
    P.b += i0 * M;
    P.Rpp += i0 * M * M;
    P.sigma_ab += i0;
    P.tau_aa += i0;
    P.sigma_bx += off;
    P.tau_ax += off;
    P.tau_xx += off;
    const bool fuse = g.prem != 0;
    if (!fuse) c->launched(launch_slots(cs, P, false, true, opt->eps_var));
    AccelArgs A = afull;
    if (fuse) set_fused(c, A, i0, J, M, false);
    A.nb = Ic;
    A.sigma_ab += i0;
    A.tau_aa += i0;
    A.sigma_bx += off;
    A.tau_ax += off;
    A.tau_xx += off;
    A.lambda += i0;
    A.lambda_in += i0;
    if (colmajor) {
      A.r_h = t1 + i0;
      A.r_u = t2 + i0;
      A.r_h_in = A.r_h;
      A.r_u_in = A.r_u;
      A.ld_p = I;
    } else {
      A.r_h += off;
      A.r_u += off;
      A.r_h_in += off;
      A.r_u_in += off;
    }
    CK(cudaEventRecord(c->evt[2 * ch], cs));
    if (opt->iters > 0) c->launched(launch_accel(cs, A, g));
    CK(cudaEventRecord(c->evt[2 * ch + 1], cs));
    if (!colmajor) {
      c->launched(launch_to_ij(cs, c->rh.as<double>() + off, t1 + i0, 1, Ic, J, I));
      c->launched(launch_to_ij(cs, c->ru.as<double>() + off, t2 + i0, 1, Ic, J, I));
    }
    // the output is I x J col-major, so a bin range is a strided row block: all
    // but the last segment go out as 2D copies on their own stream while the
    // remaining chunks upload and compute (PCIe is full duplex)
    const int sg = seg_of(ch);
    if (nseg > 1 && sg < nseg - 1 && seg_of(ch + 1) != sg) {
      const int64_t s0 = I * seg_first(sg) / nch;
      CK(cudaEventRecord(c->evx[kMaxChunks + 4], cs));
      CK(cudaStreamWaitEvent(cd, c->evx[kMaxChunks + 4], 0));
      send_rows(cd, s0, i1);
      d_done = i1;
    }
  }
  if (d_done == 0 && ldh == I) {
    CK(cudaMemcpyAsync(out->r_h, t1, S * sizeof(double), cudaMemcpyDeviceToHost, cs));
    CK(cudaMemcpyAsync(out->r_u, t2, S * sizeof(double), cudaMemcpyDeviceToHost, cs));
  } else {
    send_rows(cs, d_done, I);
  }
  CK(cudaMemcpyAsync(out->lambda, c->lam.p, I * sizeof(double), cudaMemcpyDeviceToHost, cs));
  CK(cudaEventRecord(c->evx[2], cs));
  CK(cudaStreamWaitEvent(c->stream, c->evx[2], 0));
  CK(cudaEventRecord(c->evx[kMaxChunks + 5], cd));
  CK(cudaStreamWaitEvent(c->stream, c->evx[kMaxChunks + 5], 0));
  CK(cudaEventRecord(c->ev1, c->stream));
  const auto th1 = std::chrono::steady_clock::now();
  check_err(c, J);
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  if (std::getenv("RCSCM_DEBUG_TIMING"))
    std::fprintf(stderr, "run_accel_pipelined: host enqueue %.1f us, device %.1f us, total %.1f us\n",
                 std::chrono::duration<double, std::micro>(th1 - th0).count(), ms * 1e3,
                 std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - th0).count());
  // iter_seconds (include/rcscm_gpu.h): CUDA-event time of the iteration
  // kernels only -- the sum of the chunks' K2 launches, without the copies
  double k2_ms = 0.0;
  for (int ch = 0; ch < nch; ++ch) {
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, c->evt[2 * ch], c->evt[2 * ch + 1]));
    k2_ms += t;
  }
  if (std::getenv("RCSCM_DEBUG_TIMING"))
    std::fprintf(stderr, "run_accel_pipelined: K2 launches %.1f us of the %.1f us call\n", k2_ms * 1e3, ms * 1e3);
  secs->assign(opt->iters, opt->iters ? (k2_ms * 1e-3) / opt->iters : 0.0);
  return true;
}

// Shared driver of run_naive / run_algorithm2 (solver_naive.hpp:412-450,
// solver_accel.hpp:183-240).
enum Backend { kNaive = 0, kAccel1 = 1, kAccel2 = 2 };

void run_solver(rcscm_gpu_ctx* c, Backend backend, const rcscm_inputs* in, const rcscm_params* p0,
                const rcscm_hyper* hyper, const double* X, const rcscm_solver_opts* opt, rcscm_params* out,
                rcscm_result* extra) {
  const bool accel = backend == kAccel2;  // Algorithm 2: sigma / tau precompute, K2
  const char* who = backend == kNaive ? "run_naive" : "run_accelerated";
  validate_opts(opt, who);
  validate_inputs(in, !accel || opt->compute_objective, accel);
  if (!p0 || !out || !hyper) fail(RCSCM_INVALID_INPUT, std::string(who) + ": params / hyper must not be NULL");
  const int64_t I = in->num_bins, J = in->frames;
  const int M = in->mics;
  const int iters = opt->iters;
  if (extra) {
    if (extra->n_objective) *extra->n_objective = 0;
    if (extra->n_iters) *extra->n_iters = 0;
  }
  if (I == 0) return;
  const bool traj = extra && opt->record_trajectory && (extra->traj_r_h || extra->traj_r_u || extra->traj_lambda);
  const bool fp = accel && f32(c);  // complex64 (FP32) accelerated solve
  if (fp && traj) fail(RCSCM_UNSUPPORTED, "record_trajectory is not supported in the complex64 mode");
  if (accel && !fp && !opt->compute_objective && !traj) {
    std::vector<double> secs;
    if (run_accel_pipelined(c, in, p0, hyper, X, opt, out, &secs)) {
      if (extra) {
        if (extra->iter_seconds) std::memcpy(extra->iter_seconds, secs.data(), secs.size() * sizeof(double));
        if (extra->n_iters) *extra->n_iters = opt->iters;
      }
      return;
    }
  }
  upload_model(c, in, p0, X, !accel || opt->compute_objective, accel);
  reset_err(c);
  const size_t S = static_cast<size_t>(I * J);
  if (fp) {
    alloc_f32(c, I, J, M);
    x_to_f32(c, S, M);
    params_to_f32(c, S, c->rh.as<double>(), c->ru.as<double>());
    precompute(c, problem(c, 1, I, J, M), opt->eps_var);
    // the objective is evaluated in double from the double sigma / tau
    if (opt->compute_objective) c->launched(launch_slots(c->stream, problem(c, 1, I, J, M), false, true, opt->eps_var));
  } else if (accel) {
    c->launched(launch_slots(c->stream, problem(c, 1, I, J, M), false, true, opt->eps_var));
  }
  double* trh = traj ? c->traj_rh.get<double>(S * std::max(iters, 1)) : nullptr;
  double* tru = traj ? c->traj_ru.get<double>(S * std::max(iters, 1)) : nullptr;
  double* trl = traj ? c->traj_lam.get<double>(I * std::max(iters, 1)) : nullptr;
  std::vector<double> objv, secs;
  int iters_run = 0;
  auto launch = [&](int first, int count) {
    if (backend == kAccel1) {
      Accel1Args A = accel1_args(c, I, J, count, *hyper, opt->eps_var, opt->gamma_fault);
      if (traj) {
        A.traj_r_h = trh + static_cast<size_t>(first) * S;
        A.traj_r_u = tru + static_cast<size_t>(first) * S;
        A.traj_lambda = trl + static_cast<size_t>(first) * I;
      }
      c->launched(launch_accel1(c->stream, M, A));
    } else if (accel) {
      AccelArgs A = accel_args(c, I, J, M, count, *hyper, opt->eps_var, opt->gamma_fault);
      if (traj) {
        A.traj_r_h = trh + static_cast<size_t>(first) * S;
        A.traj_r_u = tru + static_cast<size_t>(first) * S;
        A.traj_lambda = trl + static_cast<size_t>(first) * I;
      }
      run_accel(c, A);
    } else {
      NaiveArgs N = naive_args(c, I, J, count, *hyper, opt->eps_var);
      if (traj) {
        N.traj_r_h = trh + static_cast<size_t>(first) * S;
        N.traj_r_u = tru + static_cast<size_t>(first) * S;
        N.traj_lambda = trl + static_cast<size_t>(first) * I;
      }
      c->launched(launch_naive(c->stream, M, N));
    }
  };
  if (!opt->compute_objective) {
    CK(cudaEventRecord(c->ev0, c->stream));
    if (iters > 0) launch(0, iters);
    CK(cudaEventRecord(c->ev1, c->stream));
    iters_run = iters;
    check_err(c, J);
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    // one launch runs every iteration on-chip: each gets the mean time
    secs.assign(iters, iters ? (ms * 1e-3) / iters : 0.0);
  } else {
    // accel: the O(1)-per-slot objective (scalar expansion, needs log pdet R');
    // naive: the per-slot Cholesky form of model.hpp:129-157.
    if (accel) c->launched(launch_logpdet(c->stream, problem(c, 1, I, J, M)));
    if (accel && !fp && !(opt->rel_obj_tol > 0.0) && choose_accel_cfg(J).cl) {
      // no early stop: every iteration and its objective in one K2 launch
      double* dobj = c->obj.get<double>(static_cast<size_t>(iters) + 1);
      objective_fast(c, I, J, M, *hyper, dobj);
      CK(cudaEventRecord(c->ev0, c->stream));
      run_accel_obj(c, I, J, M, iters, *hyper, opt->eps_var, opt->gamma_fault, dobj, trh, tru, trl);
      CK(cudaEventRecord(c->ev1, c->stream));
      objv.resize(static_cast<size_t>(iters) + 1);
      d2h(c, objv.data(), dobj, objv.size() * sizeof(double));
      check_err(c, J);
      iters_run = iters;
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
      secs.assign(iters, iters ? (ms * 1e-3) / iters : 0.0);
    }
    auto eval = [&] {
      if (fp) params_from_f32(c, S);
      return accel ? objective_fast(c, I, J, M, *hyper) : objective(c, I, J, M, *hyper);
    };
    if (objv.empty()) objv.push_back(eval());
    for (int it = iters_run; it < iters; ++it) {
      CK(cudaEventRecord(c->ev0, c->stream));
      launch(it, 1);
      CK(cudaEventRecord(c->ev1, c->stream));
      ++iters_run;
      objv.push_back(eval());  // synchronizes + checks errors
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
      secs.push_back(ms * 1e-3);
      const double prev = objv[objv.size() - 2], cur = objv.back();
      if (opt->rel_obj_tol > 0.0 && std::abs(cur - prev) <= opt->rel_obj_tol * std::abs(prev)) break;
    }
  }
  if (fp) params_from_f32(c, S);
  download_params(c, I, J, out);
  if (traj && iters_run > 0) {
    double* th = c->tmp.get<double>(S * iters_run);
    if (extra->traj_r_h) {
      c->launched(launch_to_ij(c->stream, trh, th, iters_run, I, J));
      d2h(c, extra->traj_r_h, th, S * iters_run * sizeof(double));
    }
    if (extra->traj_r_u) {
      c->launched(launch_to_ij(c->stream, tru, th, iters_run, I, J));
      d2h(c, extra->traj_r_u, th, S * iters_run * sizeof(double));
    }
    d2h(c, extra->traj_lambda, trl, static_cast<size_t>(I) * iters_run * sizeof(double));
  }
  sync(c);
  if (extra) {
    if (extra->objective) std::memcpy(extra->objective, objv.data(), objv.size() * sizeof(double));
    if (extra->n_objective) *extra->n_objective = static_cast<int>(objv.size());
    if (extra->iter_seconds) std::memcpy(extra->iter_seconds, secs.data(), secs.size() * sizeof(double));
    if (extra->n_iters) *extra->n_iters = iters_run;
  }
}

void extract_impl(rcscm_gpu_ctx* c, const rcscm_inputs* in, const rcscm_params* p, const double* X, double* image,
                  double* dry, double* noise) {
  if (!c || !p) fail(RCSCM_INVALID_INPUT, "extract: NULL argument");
  validate_inputs(in, false, true);
  const int64_t I = in->num_bins, J = in->frames;
  const int M = in->mics;
  if (I == 0) return;
  upload_model(c, in, p, X, false, true);
  const size_t S = static_cast<size_t>(I * J);
  if (f32(c) && !noise) {
    // complex64 mode: single-precision Wiener filter from the complex64 x
    alloc_f32(c, I, J, M);
    x_to_f32(c, S, M);
    params_to_f32(c, S, c->rh.as<double>(), c->ru.as<double>());
    WienerArgsF32 Wf{};
    Wf.nb = I;
    Wf.J = J;
    Wf.X = c->Xf.as<float2>();
    Wf.a = c->a.as<double2>();
    Wf.b = c->b.as<double2>();
    Wf.Rpp = c->Rpp.as<double2>();
    Wf.r_h = c->rhf.as<float>();
    Wf.r_u = c->ruf.as<float>();
    Wf.lambda = c->lam.as<double>();
    Wf.dry = dry ? c->dryf.get<float2>(S) : nullptr;
    Wf.image = image ? c->imagef.get<float2>(S * M) : nullptr;
    c->launched(launch_wiener_f32(c->stream, M, Wf, true));
    if (dry) {
      double2* dd = c->dry.get<double2>(S);
      c->launched(launch_f2d(c->stream, c->dryf.as<float>(), reinterpret_cast<double*>(dd), 2 * S));
      double2* t = c->tmp.get<double2>(S);
      c->launched(launch_to_ij_c(c->stream, dd, t, 1, I, J));
      d2h_ij(c, dry, t, I, J, sizeof(double2));
    }
    if (image) {
      double2* im = c->image.get<double2>(S * M);
      c->launched(launch_f2d(c->stream, c->imagef.as<float>(), reinterpret_cast<double*>(im), 2 * S * M));
      d2h(c, image, im, S * M * sizeof(double2));
    }
    sync(c);
    return;
  }
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
  Wa.dry = dry ? c->dry.get<double2>(S) : nullptr;
  Wa.image = image ? c->image.get<double2>(S * M) : nullptr;
  if (noise) Wa.noise = c->noise.get<double2>(S * M);
  c->launched(launch_wiener(c->stream, M, Wa, true, noise != nullptr));
  if (dry) {
    double2* t = c->tmp.get<double2>(S);
    c->launched(launch_to_ij_c(c->stream, Wa.dry, t, 1, I, J));
    d2h_ij(c, dry, t, I, J, sizeof(double2));
  }
  if (image) d2h(c, image, Wa.image, S * M * sizeof(double2));
  if (noise) d2h(c, noise, Wa.noise, S * M * sizeof(double2));
  sync(c);
}

// ---- multi-device: contiguous bin ranges, one host thread per device ---------------
// Runs body(ctx, d, lo, hi) for device d's balanced bin range [lo, hi) of I bins
// on its own thread, with the context's ldh / bin_offset set for the range; the
// first failing range (in device order) is rethrown on the caller's thread.
template <class F>
void run_sharded(rcscm_gpu_ctx* c, int64_t I, F&& body) {
  std::vector<rcscm_gpu_ctx*> ctxs{c};
  ctxs.insert(ctxs.end(), c->peers.begin(), c->peers.end());
  const int64_t D = static_cast<int64_t>(ctxs.size());
  std::vector<ApiError> errs(ctxs.size(), ApiError{RCSCM_OK, ""});
  std::vector<std::thread> th;
  for (int64_t d = 0; d < D; ++d) {
    const int64_t lo = I * d / D, hi = I * (d + 1) / D;
    if (hi == lo) continue;
    th.emplace_back([&, d, lo, hi] {
      rcscm_gpu_ctx* x = ctxs[d];
      try {
        CK(cudaSetDevice(x->device));
        x->ldh = I;
        x->bin_offset = lo;
        struct Reset {
          rcscm_gpu_ctx* x;
          ~Reset() { x->ldh = x->bin_offset = 0; }
        } reset{x};
        body(x, d, lo, hi);
      } catch (const ApiError& e) {
        errs[d] = e;
      } catch (const std::exception& e) {
        errs[d] = ApiError{RCSCM_CUDA_ERROR, e.what()};
      }
    });
  }
  for (auto& t : th) t.join();
  CK(cudaSetDevice(c->device));
  for (const ApiError& e : errs)
    if (e.code != RCSCM_OK) fail(e.code, e.msg);
}

// rcscm_inputs / X views of bins [lo, hi)
rcscm_inputs slice_inputs(const rcscm_inputs* in, int64_t lo, int64_t hi) {
  rcscm_inputs v = *in;
  const int64_t M = in->mics;
  v.num_bins = hi - lo;
  v.a = in->a ? in->a + 2 * lo * M : nullptr;
  v.b = in->b ? in->b + 2 * lo * M : nullptr;
  v.R_prime = in->R_prime ? in->R_prime + 2 * lo * M * M : nullptr;
  v.R_prime_pinv = in->R_prime_pinv ? in->R_prime_pinv + 2 * lo * M * M : nullptr;
  return v;
}

void run_solver_sharded(rcscm_gpu_ctx* c, Backend backend, const rcscm_inputs* in, const rcscm_params* p0,
                        const rcscm_hyper* hyper, const double* X, const rcscm_solver_opts* opt, rcscm_params* out,
                        rcscm_result* extra) {
  const char* who = backend == kNaive ? "run_naive" : "run_accelerated";
  validate_opts(opt, who);
  validate_inputs(in, backend != kAccel2, backend == kAccel2);
  if (!p0 || !out || !hyper || !X) fail(RCSCM_INVALID_INPUT, std::string(who) + ": NULL argument");
  if (opt->compute_objective || opt->record_trajectory)
    fail(RCSCM_UNSUPPORTED, std::string(who) + ": compute_objective / record_trajectory run on one device");
  const int64_t I = in->num_bins, J = in->frames, M = in->mics;
  const int n = std::max(opt->iters, 0);
  std::vector<std::vector<double>> secs(1 + c->peers.size(), std::vector<double>(n, 0.0));
  run_sharded(c, I, [&](rcscm_gpu_ctx* x, int64_t d, int64_t lo, int64_t hi) {
    const rcscm_inputs v = slice_inputs(in, lo, hi);
    const rcscm_params pin{p0->r_h + lo, p0->r_u + lo, p0->lambda + lo};
    rcscm_params pout{out->r_h + lo, out->r_u + lo, out->lambda + lo};
    int nit = 0;
    rcscm_result r{nullptr, nullptr, secs[d].data(), &nit, nullptr, nullptr, nullptr};
    run_solver(x, backend, &v, &pin, hyper, X + 2 * lo * J * M, opt, &pout, &r);
  });
  if (extra) {
    if (extra->n_objective) *extra->n_objective = 0;
    if (extra->iter_seconds)  // the devices run concurrently: the slowest one's time
      for (int k = 0; k < n; ++k) {
        double m = 0.0;
        for (const auto& v : secs) m = std::max(m, v[k]);
        extra->iter_seconds[k] = m;
      }
    if (extra->n_iters) *extra->n_iters = n;
  }
}

void extract_sharded(rcscm_gpu_ctx* c, const rcscm_inputs* in, const rcscm_params* p, const double* X, double* image,
                     double* dry, double* noise) {
  if (!p || !X) fail(RCSCM_INVALID_INPUT, "extract: NULL argument");
  validate_inputs(in, false, true);
  const int64_t I = in->num_bins, J = in->frames, M = in->mics;
  run_sharded(c, I, [&](rcscm_gpu_ctx* x, int64_t, int64_t lo, int64_t hi) {
    const rcscm_inputs v = slice_inputs(in, lo, hi);
    const rcscm_params pv{p->r_h + lo, p->r_u + lo, p->lambda + lo};
    const size_t o = static_cast<size_t>(2 * lo * J * M);
    extract_impl(x, &v, &pv, X + o, image ? image + o : nullptr, dry ? dry + 2 * lo : nullptr,
                 noise ? noise + o : nullptr);
  });
}

}  // namespace rcscm_capi

// =============================================================================
// C ABI
// =============================================================================
extern "C" {

const char* rcscm_gpu_last_error(void) { return g_last_error.c_str(); }

// One context on `device` (stream: the caller's, or a context-owned one).
static rcscm_gpu_ctx* make_ctx(int device, int precision, void* stream) {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) fail(RCSCM_INVALID_INPUT, "device ordinal out of range");
  CK(cudaSetDevice(device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    fail(RCSCM_UNSUPPORTED, std::string("this build targets sm_100a (B200); device is ") + prop.name);
  auto* c = new rcscm_gpu_ctx();
  c->device = device;
  c->precision = precision;
  try {
    if (stream) {
      c->stream = static_cast<cudaStream_t>(stream);
    } else {
      CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    CK(cudaEventCreate(&c->ev0));
    CK(cudaEventCreate(&c->ev1));
  } catch (...) {
    rcscm_gpu_destroy(c);
    throw;
  }
  return c;
}

int rcscm_gpu_create(const rcscm_gpu_config* cfg, rcscm_gpu_ctx** out) {
  return guarded([&] {
    if (!out) fail(RCSCM_INVALID_INPUT, "out must not be NULL");
    *out = nullptr;
    rcscm_gpu_config d{0, RCSCM_C128, nullptr, nullptr, 0};
    if (cfg) d = *cfg;
    if (d.precision != RCSCM_C128 && d.precision != RCSCM_C64) fail(RCSCM_INVALID_INPUT, "precision must be RCSCM_C128 or RCSCM_C64");
    if (d.num_devices < 0 || (d.num_devices > 1 && !d.devices))
      fail(RCSCM_INVALID_INPUT, "create: devices must list num_devices ordinals");
    const int nd = d.num_devices > 1 ? d.num_devices : 1;
    const int dev0 = (d.num_devices >= 1 && d.devices) ? d.devices[0] : d.device;
    rcscm_gpu_ctx* c = make_ctx(dev0, d.precision, d.stream);
    try {
      for (int k = 1; k < nd; ++k) c->peers.push_back(make_ctx(d.devices[k], d.precision, nullptr));
    } catch (...) {
      rcscm_gpu_destroy(c);
      throw;
    }
    CK(cudaSetDevice(dev0));
    *out = c;
  });
}

void rcscm_gpu_destroy(rcscm_gpu_ctx* c) {
  if (!c) return;
  for (rcscm_gpu_ctx* p : c->peers) rcscm_gpu_destroy(p);
  c->peers.clear();
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (DBuf* b : {&c->X, &c->W, &c->A, &c->T, &c->V, &c->a, &c->b, &c->Rp, &c->Rpp, &c->power, &c->sab, &c->taa,
                  &c->sbx, &c->tax, &c->txx, &c->rh, &c->ru, &c->lam, &c->lpd, &c->rh0, &c->ru0, &c->lam0, &c->tmp,
                  &c->tmp2, &c->traj_rh, &c->traj_ru, &c->traj_lam, &c->scratch, &c->gam, &c->dry, &c->image, &c->noise,
                  &c->partial, &c->obj, &c->obj_part, &c->err, &c->Xf, &c->sbxf, &c->taxf, &c->txxf, &c->rhf, &c->ruf,
                  &c->dryf, &c->imagef, &c->rh0f, &c->ru0f, &c->st_x, &c->st_w, &c->st_f, &c->st_spec, &c->st_part,
                  &c->st_lam,
                  &c->st_X, &c->il_X, &c->il_W, &c->il_A, &c->il_T, &c->il_V, &c->il_P, &c->il_part, &c->il_mu, &c->il_Pt, &c->il_ucov,
                  &c->ex_Q, &c->ex_W, &c->ex_A, &c->ex_pow, &c->ex_out, &c->ex_obj})
    b->release();
  c->ex_pin.release();
  c->err_pin.release();
  if (c->il_graph) cudaGraphExecDestroy(c->il_graph);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  for (int k = 0; k < 4; ++k)
    if (c->aux[k]) cudaStreamDestroy(c->aux[k]);
  for (cudaEvent_t e : c->evx)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : c->evt)
    if (e) cudaEventDestroy(e);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
}

int64_t rcscm_gpu_launch_count(const rcscm_gpu_ctx* c) {
  if (!c) return 0;
  int64_t n = c->launches;
  for (const rcscm_gpu_ctx* p : c->peers) n += p->launches;
  return n;
}

void* rcscm_gpu_stream(rcscm_gpu_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

int rcscm_gpu_build_noise_scm(rcscm_gpu_ctx* c, int64_t I, int64_t J, int M, const double* X, const double* W,
                              const double* A, int n_h, double rank_tol, double* a, double* Rp, double* Rpp,
                              double* b) {
  return guarded([&] {
    if (!c) fail(RCSCM_INVALID_INPUT, "ctx must not be NULL");
    if (n_h < 0 || n_h >= M) fail(RCSCM_INVALID_INPUT, "build_noise_scm: target index out of range");
    if (I < 0 || J < 0 || M < 1) fail(RCSCM_INVALID_INPUT, "build_noise_scm: bad shape");
    if (I == 0) return;
    if (J < 1) fail(RCSCM_INVALID_INPUT, "build_noise_scm: frames must be >= 1");
    check_mics(M);
    alloc_problem(c, I, J, M);
    c->W.get<double2>(I * M * M);
    c->A.get<double2>(I * M * M);
    h2d(c, c->X.p, X, static_cast<size_t>(I * J * M) * sizeof(double2));
    h2d(c, c->W.p, W, I * M * M * sizeof(double2));
    h2d(c, c->A.p, A, I * M * M * sizeof(double2));
    reset_err(c);
    c->sn_h = n_h;
    c->launched(launch_setup(c->stream, problem(c, 1, I, J, M), rank_tol, 1e-12), 2);
    check_err(c, J);
    d2h(c, a, c->a.p, I * M * sizeof(double2));
    d2h(c, b, c->b.p, I * M * sizeof(double2));
    d2h(c, Rp, c->Rp.p, I * M * M * sizeof(double2));
    d2h(c, Rpp, c->Rpp.p, I * M * M * sizeof(double2));
    sync(c);
  });
}

int rcscm_gpu_init_params(rcscm_gpu_ctx* c, const rcscm_inputs* in, int K, const double* X, const double* W,
                          const double* A, const double* T, const double* V, rcscm_params* out) {
  return guarded([&] {
    if (!c) fail(RCSCM_INVALID_INPUT, "ctx must not be NULL");
    validate_inputs(in, true, true);
    if (!out) fail(RCSCM_INVALID_INPUT, "init_params: out must not be NULL");
    const int64_t I = in->num_bins, J = in->frames;
    const int M = in->mics;
    if (in->n_h < 0 || in->n_h >= M) fail(RCSCM_INVALID_INPUT, "init_params: target index out of range");
    if (K < 0) fail(RCSCM_INVALID_INPUT, "init_params: K must be >= 0");
    if (I == 0) return;
    upload_model(c, in, nullptr, X, true, true);
    c->W.get<double2>(I * M * M);
    c->A.get<double2>(I * M * M);
    c->T.get<double>(std::max<int64_t>(I * K, 1));
    c->V.get<double>(std::max<int64_t>(K * J, 1));
    h2d(c, c->W.p, W, I * M * M * sizeof(double2));
    h2d(c, c->A.p, A, I * M * M * sizeof(double2));
    h2d(c, c->T.p, T, I * K * sizeof(double));
    h2d(c, c->V.p, V, K * J * sizeof(double));
    reset_err(c);
    c->sn_h = in->n_h;
    c->sK = K;
    DevProblem P = problem(c, 1, I, J, M);
    c->launched(launch_slots(c->stream, P, true, false, 1e-12));
    c->launched(launch_lambda0(c->stream, P, 1e-12));
    check_err(c, J);
    download_params(c, I, J, out);
    sync(c);
  });
}

int rcscm_gpu_map_objective(rcscm_gpu_ctx* c, const rcscm_inputs* in, const rcscm_params* p,
                            const rcscm_hyper* hyper, const double* X, double* out) {
  return guarded([&] {
    if (!c || !p || !hyper || !out) fail(RCSCM_INVALID_INPUT, "map_objective: NULL argument");
    validate_inputs(in, true, false);
    const int64_t I = in->num_bins, J = in->frames;
    *out = 0.0;
    if (I == 0) return;
    upload_model(c, in, p, X, true, false);
    reset_err(c);
    *out = objective(c, I, J, in->mics, *hyper);
  });
}

int rcscm_gpu_run_naive(rcscm_gpu_ctx* c, const rcscm_inputs* in, const rcscm_params* params0,
                        const rcscm_hyper* hyper, const double* X, const rcscm_solver_opts* opt, rcscm_params* out,
                        rcscm_result* extra) {
  return guarded([&] {
    if (!c) fail(RCSCM_INVALID_INPUT, "ctx must not be NULL");
    if (!c->peers.empty()) return run_solver_sharded(c, kNaive, in, params0, hyper, X, opt, out, extra);
    run_solver(c, kNaive, in, params0, hyper, X, opt, out, extra);
  });
}

int rcscm_gpu_run_algorithm2(rcscm_gpu_ctx* c, const rcscm_inputs* in, const rcscm_params* params0,
                             const rcscm_hyper* hyper, const double* X, const rcscm_solver_opts* opt,
                             rcscm_params* out, rcscm_result* extra) {
  return guarded([&] {
    if (!c) fail(RCSCM_INVALID_INPUT, "ctx must not be NULL");
    if (!c->peers.empty()) return run_solver_sharded(c, kAccel2, in, params0, hyper, X, opt, out, extra);
    run_solver(c, kAccel2, in, params0, hyper, X, opt, out, extra);
  });
}

int rcscm_gpu_run_algorithm1(rcscm_gpu_ctx* c, const rcscm_inputs* in, const rcscm_params* params0,
                             const rcscm_hyper* hyper, const double* X, const rcscm_solver_opts* opt,
                             rcscm_params* out, rcscm_result* extra) {
  return guarded([&] {
    if (!c) fail(RCSCM_INVALID_INPUT, "ctx must not be NULL");
    if (!c->peers.empty()) return run_solver_sharded(c, kAccel1, in, params0, hyper, X, opt, out, extra);
    run_solver(c, kAccel1, in, params0, hyper, X, opt, out, extra);
  });
}

int rcscm_gpu_run_accel(rcscm_gpu_ctx* c, int stage, const rcscm_inputs* in, const rcscm_params* params0,
                        const rcscm_hyper* hyper, const double* X, const rcscm_solver_opts* opt, rcscm_params* out,
                        rcscm_result* extra) {
  if (stage == 1) return rcscm_gpu_run_algorithm1(c, in, params0, hyper, X, opt, out, extra);
  if (stage == 2) return rcscm_gpu_run_algorithm2(c, in, params0, hyper, X, opt, out, extra);
  return guarded([&] { fail(RCSCM_INVALID_INPUT, "run_accel: stage must be 1 or 2, got " + std::to_string(stage)); });
}

int rcscm_gpu_build_inputs(rcscm_gpu_ctx* c, int64_t I, int64_t J, int M, const double* X, const double* W,
                           const double* A, int n_h, double rank_tol, int K, const double* T, const double* V,
                           double* a, double* R_prime, double* R_prime_pinv, double* b, rcscm_params* out) {
  // build_noise_scm then init_params (model.hpp:58-124) on the device buffers the
  // setup kernel leaves resident: x, W and A go up once, only the requested
  // outputs come back (any of a / R' / R'^+ / b may be NULL)
  return guarded([&] {
    if (!c) fail(RCSCM_INVALID_INPUT, "ctx must not be NULL");
    // (with a device list the setup runs on devices[0]; sharding is for the solvers)
    if (n_h < 0 || n_h >= M) fail(RCSCM_INVALID_INPUT, "build_noise_scm: target index out of range");
    if (I < 0 || J < 0 || M < 1) fail(RCSCM_INVALID_INPUT, "build_noise_scm: bad shape");
    if (K < 0) fail(RCSCM_INVALID_INPUT, "init_params: K must be >= 0");
    if (!out) fail(RCSCM_INVALID_INPUT, "init_params: out must not be NULL");
    if (I == 0) return;
    if (J < 1) fail(RCSCM_INVALID_INPUT, "build_noise_scm: frames must be >= 1");
    check_mics(M);
    alloc_problem(c, I, J, M);
    c->W.get<double2>(I * M * M);
    c->A.get<double2>(I * M * M);
    c->T.get<double>(std::max<int64_t>(I * K, 1));
    c->V.get<double>(std::max<int64_t>(K * J, 1));
    h2d(c, c->X.p, X, static_cast<size_t>(I * J * M) * sizeof(double2));
    h2d(c, c->W.p, W, I * M * M * sizeof(double2));
    h2d(c, c->A.p, A, I * M * M * sizeof(double2));
    h2d(c, c->T.p, T, I * K * sizeof(double));
    h2d(c, c->V.p, V, K * J * sizeof(double));
    reset_err(c);
    c->sn_h = n_h;
    c->sK = K;
    const DevProblem P = problem(c, 1, I, J, M);
    c->launched(launch_setup(c->stream, P, rank_tol, kEpsVar), 2);
    check_err(c, J);  // build_noise_scm's errors first, as the two calls report them
    c->launched(launch_slots(c->stream, P, true, false, kEpsVar));
    c->launched(launch_lambda0(c->stream, P, kEpsVar));
    check_err(c, J);
    d2h(c, a, c->a.p, I * M * sizeof(double2));
    d2h(c, b, c->b.p, I * M * sizeof(double2));
    d2h(c, R_prime, c->Rp.p, I * M * M * sizeof(double2));
    d2h(c, R_prime_pinv, c->Rpp.p, I * M * M * sizeof(double2));
    download_params(c, I, J, out);
    sync(c);
  });
}

int rcscm_gpu_extract_target(rcscm_gpu_ctx* c, const rcscm_inputs* in, const rcscm_params* p, const double* X,
                             double* image, double* dry) {
  return guarded([&] {
    if (c && !c->peers.empty()) return extract_sharded(c, in, p, X, image, dry, nullptr);
    extract_impl(c, in, p, X, image, dry, nullptr);
  });
}

int rcscm_gpu_extract_noise(rcscm_gpu_ctx* c, const rcscm_inputs* in, const rcscm_params* p, const double* X,
                            double* noise) {
  return guarded([&] {
    if (!noise) fail(RCSCM_INVALID_INPUT, "extract_noise: noise must not be NULL");
    if (c && !c->peers.empty()) return extract_sharded(c, in, p, X, nullptr, nullptr, noise);
    extract_impl(c, in, p, X, nullptr, nullptr, noise);
  });
}

}  // extern "C"

// session_load from host (H2D) or device (D2D) buffers
void rcscm_capi::session_load_impl(rcscm_gpu_ctx* c, int64_t B, int64_t I, int64_t J, int M, int K, int n_h,
                              const void* X, const void* W, const void* A, const void* T, const void* V,
                              cudaMemcpyKind kind) {
    if (!c) fail(RCSCM_INVALID_INPUT, "ctx must not be NULL");
    if (B < 1 || I < 1 || J < 1 || M < 1 || K < 0) fail(RCSCM_INVALID_INPUT, "session_load: bad shape");
    if (n_h < 0 || n_h >= M) fail(RCSCM_INVALID_INPUT, "session_load: target index out of range");
    check_mics(M);
    const int64_t nb = B * I;
    alloc_problem(c, nb, J, M);
    c->W.get<double2>(nb * M * M);
    c->A.get<double2>(nb * M * M);
    c->T.get<double>(std::max<int64_t>(B * I * K, 1));
    c->V.get<double>(std::max<int64_t>(B * K * J, 1));
    const size_t S = static_cast<size_t>(nb * J);
    c->rh0.get<double>(S);
    c->ru0.get<double>(S);
    c->lam0.get<double>(nb);
    c->dry.get<double2>(S);
    c->image.get<double2>(S * M);
    c->scratch.get<double2>(S);
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      if (bytes && dst != src) CK(cudaMemcpyAsync(dst, src, bytes, kind, c->stream));
    };
    cp(c->X.p, X, S * M * sizeof(double2));
    cp(c->W.p, W, nb * M * M * sizeof(double2));
    cp(c->A.p, A, nb * M * M * sizeof(double2));
    cp(c->T.p, T, B * I * K * sizeof(double));
    cp(c->V.p, V, B * K * J * sizeof(double));
    if (f32(c)) {
      alloc_f32(c, nb, J, M);
      c->dryf.get<float2>(S);
      c->imagef.get<float2>(S * M);
      x_to_f32(c, S, M);
    }
    c->f32_params_current = false;
    c->sB = B;
    c->sI = I;
    c->sJ = J;
    c->sM = M;
    c->sK = K;
    c->sn_h = n_h;
    c->s_loaded = true;
    c->s_setup = false;
    c->s_pre = false;
    c->s_reset_pending = false;
    reset_err(c);
    sync(c);
}

extern "C" {

int rcscm_gpu_session_load(rcscm_gpu_ctx* c, int64_t B, int64_t I, int64_t J, int M, int K, int n_h, const double* X,
                           const double* W, const double* A, const double* T, const double* V) {
  return guarded([&] { session_load_impl(c, B, I, J, M, K, n_h, X, W, A, T, V, cudaMemcpyHostToDevice); });
}

// Applies a pending RESET to the working iterate (rh, ru, lam and the FP32 copies).
static void materialize_reset(rcscm_gpu_ctx* c, size_t S, int64_t nb) {
  if (!c->s_reset_pending) return;
  d2d(c, c->rh.p, c->rh0.p, S * sizeof(double));
  d2d(c, c->ru.p, c->ru0.p, S * sizeof(double));
  d2d(c, c->lam.p, c->lam0.p, nb * sizeof(double));
  if (f32(c)) {
    d2d(c, c->rhf.p, c->rh0f.p, S * sizeof(float));
    d2d(c, c->ruf.p, c->ru0f.p, S * sizeof(float));
    c->f32_params_current = true;
  }
  c->s_reset_pending = false;
}

int rcscm_gpu_session_run(rcscm_gpu_ctx* c, int stages, int iters, const rcscm_hyper* hyper, double eps_var) {
  return guarded([&] {
    if (!c || !c->s_loaded) fail(RCSCM_INVALID_INPUT, "session_run: no session loaded");
    if (iters < 0) fail(RCSCM_INVALID_INPUT, "session_run: iters must be >= 0");
    const rcscm_hyper h = hyper ? *hyper : rcscm_hyper{1.1, 1e-16};
    const int64_t nb = c->sB * c->sI, J = c->sJ;
    const int M = c->sM;
    const size_t S = static_cast<size_t>(nb * J);
    DevProblem P = problem(c, c->sB, c->sI, J, M);
    bool pre_done = false;
    // PRECOMPUTE + ACCEL in one call (complex128, tuned K2 shape): one fused kernel
    // forms sigma / tau from x in K2's prologue (and keeps them for WIENER)
    const bool fuse_pre = (stages & RCSCM_STAGE_PRECOMPUTE) && (stages & RCSCM_STAGE_ACCEL) &&
                          !(stages & RCSCM_STAGE_SETUP) && !f32(c) && accel_fusable(choose_accel_cfg(J), M);
    const char* e_fw = std::getenv("RCSCM_FUSE_WIENER");  // 0: K4 after K2 (A/B knob)
    const bool fuse_wiener = fuse_pre && (stages & RCSCM_STAGE_WIENER) && !(stages & RCSCM_STAGE_NAIVE) &&
                             iters > 0 && !(e_fw && std::atoi(e_fw) == 0);
    if (stages & RCSCM_STAGE_SETUP) {
      // init_params floors r_h0, r_u0 and lambda0 with kEpsVar (model.hpp:102,110,121),
      // whatever eps_var the solver stages use
      c->launched(launch_setup(c->stream, P, 1e-10, kEpsVar), 2);
      const bool pre = (stages & RCSCM_STAGE_PRECOMPUTE) != 0 && !f32(c);
      c->launched(launch_slots(c->stream, P, true, pre, kEpsVar));
      pre_done = pre;
      if (f32(c)) {
        params_to_f32(c, S, c->rh.as<double>(), c->ru.as<double>());
        c->f32_params_current = true;
        d2d(c, c->rh0f.get<float>(S), c->rhf.p, S * sizeof(float));
        d2d(c, c->ru0f.get<float>(S), c->ruf.p, S * sizeof(float));
      }
      d2d(c, c->rh0.p, c->rh.p, S * sizeof(double));
      d2d(c, c->ru0.p, c->ru.p, S * sizeof(double));
      d2d(c, c->lam0.p, c->lam.p, nb * sizeof(double));
      c->s_setup = true;
      c->s_reset_pending = false;
      if (pre) c->s_pre = true;
    }
    if (!c->s_setup) fail(RCSCM_INVALID_INPUT, "session_run: run RCSCM_STAGE_SETUP first");
    if (stages & RCSCM_STAGE_RESET) c->s_reset_pending = true;
    if ((stages & RCSCM_STAGE_PRECOMPUTE) && !pre_done && !fuse_pre) {
      precompute(c, P, eps_var);
      c->s_pre = true;
    }
    if (stages & RCSCM_STAGE_ACCEL) {
      if (!c->s_pre && !fuse_pre) fail(RCSCM_INVALID_INPUT, "session_run: ACCEL needs PRECOMPUTE");
      AccelArgs A = accel_args(c, nb, J, M, iters, h, eps_var, 0.0);
      // the forms depend only on the session's setup outputs: store them only
      // if no earlier precompute has (WIENER reads them)
      if (fuse_pre) set_fused(c, A, 0, J, M, !c->s_pre);
      // ACCEL then WIENER in one call: K2's epilogue writes dry / image from
      // registers (the final state is the one WIENER would read back)
      if (fuse_wiener) {
        A.dry_w = c->dry.as<double2>();
        A.image_w = c->image.as<double2>();
      }
      if (c->s_reset_pending) {
        A.r_h_in = c->rh0.as<double>();
        A.r_u_in = c->ru0.as<double>();
        A.lambda_in = c->lam0.as<double>();
        A.r_h_f_in = c->rh0f.as<float>();
        A.r_u_f_in = c->ru0f.as<float>();
        c->s_reset_pending = false;
      }
      run_accel(c, A, fuse_pre ? M : 0);
      if (fuse_pre) c->s_pre = true;
      if (f32(c)) c->f32_params_current = true;
    }
    if (stages & (RCSCM_STAGE_NAIVE | RCSCM_STAGE_WIENER)) materialize_reset(c, S, nb);
    if (stages & RCSCM_STAGE_NAIVE) {
      // the naive comparison rule runs in complex128 in both modes
      if (f32(c) && c->f32_params_current) params_from_f32(c, S);
      c->launched(launch_naive(c->stream, M, naive_args(c, nb, J, iters, h, eps_var)));
      c->f32_params_current = false;
    }
    if ((stages & RCSCM_STAGE_WIENER) && !fuse_wiener) {
      if (!c->s_pre) fail(RCSCM_INVALID_INPUT, "session_run: WIENER needs PRECOMPUTE");
      WienerArgs Wa{};
      Wa.nb = nb;
      Wa.J = J;
      Wa.a = c->a.as<double2>();
      Wa.sigma_ab = c->sab.as<double2>();
      Wa.tau_aa = c->taa.as<double>();
      Wa.sigma_bx = c->sbx.as<double2>();
      Wa.tau_ax = c->tax.as<double2>();
      Wa.r_h = c->rh.as<double>();
      Wa.r_u = c->ru.as<double>();
      Wa.lambda = c->lam.as<double>();
      Wa.dry = c->dry.as<double2>();
      Wa.image = c->image.as<double2>();
      if (f32(c)) {
        if (!c->f32_params_current) params_to_f32(c, S, c->rh.as<double>(), c->ru.as<double>());
        WienerArgsF32 Wf{};
        Wf.nb = nb;
        Wf.J = J;
        Wf.a = Wa.a;
        Wf.sigma_ab = Wa.sigma_ab;
        Wf.tau_aa = Wa.tau_aa;
        Wf.sigma_bx = c->sbxf.as<float2>();
        Wf.tau_ax = c->taxf.as<float2>();
        Wf.r_h = c->rhf.as<float>();
        Wf.r_u = c->ruf.as<float>();
        Wf.lambda = Wa.lambda;
        Wf.dry = c->dryf.as<float2>();
        Wf.image = c->imagef.as<float2>();
        c->launched(launch_wiener_f32(c->stream, M, Wf, false));
        c->launched(launch_f2d(c->stream, c->dryf.as<float>(), c->dry.as<double>(), 2 * S));
        c->launched(launch_f2d(c->stream, c->imagef.as<float>(), c->image.as<double>(), 2 * S * M));
      } else {
        c->launched(launch_wiener(c->stream, M, Wa, false, false));
      }
    }
  });
}

int rcscm_gpu_session_fetch(rcscm_gpu_ctx* c, double* r_h, double* r_u, double* lambda, double* dry, double* image,
                            int do_sync) {
  return guarded([&] {
    if (!c || !c->s_loaded) fail(RCSCM_INVALID_INPUT, "session_fetch: no session loaded");
    const int64_t nb = c->sB * c->sI, J = c->sJ;
    const size_t S = static_cast<size_t>(nb * J);
    materialize_reset(c, S, nb);
    if (f32(c) && c->f32_params_current) params_from_f32(c, S);
    // host or device destinations (unified addressing decides the direction):
    // a multi-GPU caller fetches straight into its transfer tensors for the gather
    auto out = [&](void* dst, const void* src, size_t bytes) {
      if (dst && bytes) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->stream));
    };
    out(r_h, c->rh.p, S * sizeof(double));
    out(r_u, c->ru.p, S * sizeof(double));
    out(lambda, c->lam.p, nb * sizeof(double));
    out(dry, c->dry.p, S * sizeof(double2));
    out(image, c->image.p, S * c->sM * sizeof(double2));
    if (do_sync) sync(c);
  });
}

int rcscm_gpu_session_check(rcscm_gpu_ctx* c) {
  return guarded([&] {
    if (!c || !c->s_loaded) fail(RCSCM_INVALID_INPUT, "session_check: no session loaded");
    check_err(c, c->sJ);
  });
}

static int probe(rcscm_gpu_ctx* c, bool fp32, double* tflops, double* ms) {
  return guarded([&] {
    if (!c || !tflops) fail(RCSCM_INVALID_INPUT, "probe: NULL argument");
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
    constexpr int kNacc = 8, kNt = 256;
    const int blocks = sms * 8, iters = fp32 ? 40000 : 20000;
    double* out = c->obj.get<double>(1);
    auto run = [&](int n) { return fp32 ? launch_fp32_probe(c->stream, blocks, n, out) : launch_fp64_probe(c->stream, blocks, n, out); };
    c->launched(run(iters / 10));  // warm-up
    CK(cudaEventRecord(c->ev0, c->stream));
    c->launched(run(iters));
    CK(cudaEventRecord(c->ev1, c->stream));
    CK(cudaEventSynchronize(c->ev1));
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, c->ev0, c->ev1));
    const double flops = 2.0 * kNacc * static_cast<double>(iters) * blocks * kNt;
    *tflops = flops / (t * 1e-3) / 1e12;
    if (ms) *ms = t;
  });
}

int rcscm_gpu_probe_fp64(rcscm_gpu_ctx* c, double* tflops, double* ms) { return probe(c, false, tflops, ms); }
int rcscm_gpu_probe_fp32(rcscm_gpu_ctx* c, double* tflops, double* ms) { return probe(c, true, tflops, ms); }

}  // extern "C"
