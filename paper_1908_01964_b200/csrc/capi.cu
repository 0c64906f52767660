// capi.cu -- host side of the rcscm B200 path: the C ABI of include/rcscm_gpu.h.
//
// Each reference entry point (model.hpp, solver_naive.hpp, solver_accel.hpp,
// wiener.hpp) becomes: host->device copies of the caller's reference-layout
// buffers, one transpose of the I x J column-major parameters into the
// device's bin-major layout, the CUDA kernels, and the way back. There is no
// CPU fallback: every numeric step runs in the kernels of setup.cuh,
// accel.cuh, naive.cuh and stream.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/rcscm_gpu.h"
#include "accel.cuh"
#include "common.cuh"
#include "naive.cuh"
#include "setup.cuh"
#include "stream.cuh"

using namespace rcscm;

namespace {

thread_local std::string g_last_error;

struct ApiError {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw ApiError{code, msg}; }

#define CK(expr)                                                                     \
  do {                                                                               \
    cudaError_t e_ = (expr);                                                         \
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

template <class F>
void dispatch_m(int M, F&& f) {
  switch (M) {
    case 1: f(std::integral_constant<int, 1>{}); break;
    case 2: f(std::integral_constant<int, 2>{}); break;
    case 3: f(std::integral_constant<int, 3>{}); break;
    case 4: f(std::integral_constant<int, 4>{}); break;
    case 5: f(std::integral_constant<int, 5>{}); break;
    case 6: f(std::integral_constant<int, 6>{}); break;
    case 7: f(std::integral_constant<int, 7>{}); break;
    case 8: f(std::integral_constant<int, 8>{}); break;
    case 16: f(std::integral_constant<int, 16>{}); break;
    default: fail(RCSCM_UNSUPPORTED, "mics = " + std::to_string(M) + " is not supported (1..8 or 16)");
  }
}

}  // namespace

struct rcscm_gpu_ctx {
  int device = 0;
  int precision = RCSCM_C128;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int64_t launches = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // device buffers
  DBuf X, W, A, T, V, a, b, Rp, Rpp, power, sab, taa, sbx, tax, txx, rh, ru, lam;
  DBuf rh0, ru0, lam0, tmp, tmp2, traj_rh, traj_ru, traj_lam, scratch, dry, image, noise, partial, obj, err;
  // session geometry
  bool s_loaded = false, s_setup = false, s_pre = false;
  int64_t sB = 0, sI = 0, sJ = 0;
  int sM = 0, sK = 0, sn_h = 0;

  void launched() {
    CK(cudaGetLastError());
    ++launches;
  }
};

namespace {

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

void h2d(rcscm_gpu_ctx* c, void* dst, const void* src, size_t bytes) {
  if (bytes) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
}
void d2h(rcscm_gpu_ctx* c, void* dst, const void* src, size_t bytes) {
  if (bytes && dst) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
}
void sync(rcscm_gpu_ctx* c) { CK(cudaStreamSynchronize(c->stream)); }

// I x J column-major (per utterance block) <-> [bin][t]
template <class T>
void to_bt(rcscm_gpu_ctx* c, const T* src, T* dst, int64_t B, int64_t I, int64_t J) {
  if (B * I * J == 0) return;
  dim3 grid((I + 31) / 32, (J + 31) / 32, B), block(32, 8);
  k_ij_to_bt<T><<<grid, block, 0, c->stream>>>(src, dst, I, J);
  c->launched();
}
template <class T>
void to_ij(rcscm_gpu_ctx* c, const T* src, T* dst, int64_t B, int64_t I, int64_t J) {
  if (B * I * J == 0) return;
  dim3 grid((I + 31) / 32, (J + 31) / 32, B), block(32, 8);
  k_bt_to_ij<T><<<grid, block, 0, c->stream>>>(src, dst, I, J);
  c->launched();
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
    default:
      *msg = "device error code " + std::to_string(code);
      return RCSCM_NUMERICAL;
  }
}

void check_err(rcscm_gpu_ctx* c, int64_t J) {
  unsigned long long key = ~0ull;
  CK(cudaMemcpyAsync(&key, c->err.as<unsigned long long>(), sizeof(key), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
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
  c->err.get<unsigned long long>(1);
}

constexpr int kSlotNT = 128;

template <int M>
void launch_slots(rcscm_gpu_ctx* c, const DevProblem& P, bool init, bool pre, double eps) {
  if (P.nb * P.J == 0) return;
  dim3 grid(P.nb, (P.J + kSlotNT - 1) / kSlotNT);
  if (init && pre)
    k_slots<M, kSlotNT, true, true><<<grid, kSlotNT, 0, c->stream>>>(P, eps);
  else if (init)
    k_slots<M, kSlotNT, true, false><<<grid, kSlotNT, 0, c->stream>>>(P, eps);
  else
    k_slots<M, kSlotNT, false, true><<<grid, kSlotNT, 0, c->stream>>>(P, eps);
  c->launched();
}

template <int M>
void launch_setup(rcscm_gpu_ctx* c, const DevProblem& P, double rank_tol, double eps) {
  if (P.nb == 0) return;
  k_setup_power<M, 256><<<P.nb, 256, 0, c->stream>>>(P);
  c->launched();
  k_setup_bin<M, 0><<<(P.nb + 63) / 64, 64, 0, c->stream>>>(P, rank_tol, eps);
  c->launched();
}

// ---- K2 launch configuration --------------------------------------------------
struct AccelCfg {
  int cl, nt, spt;
};

AccelCfg choose_accel_cfg(int64_t J) {
  AccelCfg best{0, 0, 0};
  const char* e_spt = std::getenv("RCSCM_ACCEL_SPT");
  const char* e_cl = std::getenv("RCSCM_ACCEL_CL");
  const int force_spt = e_spt ? std::atoi(e_spt) : 0;
  const int force_cl = e_cl ? std::atoi(e_cl) : 0;
  for (int cl : {1, 2, 4, 8, 16}) {
    if (force_cl && cl != force_cl) continue;
    const int64_t jc = (J + cl - 1) / cl;
    const int max_spt = (cl == 16) ? 8 : 6;
    if (jc > 256LL * (force_spt ? force_spt : max_spt)) continue;
    int64_t best_waste = -1;
    for (int spt = 1; spt <= 8; ++spt) {
      if (force_spt ? spt != force_spt : spt > max_spt) continue;
      int64_t nt = (jc + spt - 1) / spt;
      nt = (nt + 31) / 32 * 32;
      if (nt > 256) continue;
      const int64_t waste = nt * spt - jc;
      // least idle lanes; ties go to more slots per thread (ILP, fewer warps)
      if (best_waste < 0 || waste < best_waste || (waste == best_waste && spt > best.spt)) {
        best_waste = waste;
        best = AccelCfg{cl, static_cast<int>(nt), spt};
      }
    }
    if (best.cl) return best;
  }
  fail(RCSCM_UNSUPPORTED, "frames = " + std::to_string(J) + " exceeds the on-chip accel kernel capacity (16 x 2048)");
}

template <int SPT, int CL>
void launch_accel_t(rcscm_gpu_ctx* c, const AccelArgs& A, int nt) {
  auto kern = k_accel<SPT, CL>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(A.nb * CL));
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[1];
  int na = 0;
  if (CL > 1) {
    if (CL > 8) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    na = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  CK(cudaLaunchKernelEx(&cfg, kern, A));
  c->launched();
}

template <int CL>
void launch_accel_spt(rcscm_gpu_ctx* c, const AccelArgs& A, const AccelCfg& g) {
  switch (g.spt) {
    case 1: launch_accel_t<1, CL>(c, A, g.nt); break;
    case 2: launch_accel_t<2, CL>(c, A, g.nt); break;
    case 3: launch_accel_t<3, CL>(c, A, g.nt); break;
    case 4: launch_accel_t<4, CL>(c, A, g.nt); break;
    case 5: launch_accel_t<5, CL>(c, A, g.nt); break;
    case 6: launch_accel_t<6, CL>(c, A, g.nt); break;
    case 7: launch_accel_t<7, CL>(c, A, g.nt); break;
    case 8: launch_accel_t<8, CL>(c, A, g.nt); break;
    default: fail(RCSCM_UNSUPPORTED, "bad slots-per-thread");
  }
}

void launch_accel(rcscm_gpu_ctx* c, const AccelArgs& A) {
  if (A.nb * A.J == 0) return;
  const AccelCfg g = choose_accel_cfg(A.J);
  switch (g.cl) {
    case 1: launch_accel_spt<1>(c, A, g); break;
    case 2: launch_accel_spt<2>(c, A, g); break;
    case 4: launch_accel_spt<4>(c, A, g); break;
    case 8: launch_accel_spt<8>(c, A, g); break;
    case 16: launch_accel_spt<16>(c, A, g); break;
  }
}

AccelArgs accel_args(rcscm_gpu_ctx* c, int64_t nb, int64_t J, int M, int iters, const rcscm_hyper& h,
                     double eps, double gamma_fault) {
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
  return A;
}

constexpr int kNaiveNT = 128;

template <int M>
void launch_naive(rcscm_gpu_ctx* c, NaiveArgs N) {
  if (N.nb * N.J == 0) return;
  k_naive<M, kNaiveNT><<<N.nb, kNaiveNT, 0, c->stream>>>(N);
  c->launched();
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

constexpr int kWienerNT = 128;

template <int M, bool FROM_X, bool NOISE>
void launch_wiener(rcscm_gpu_ctx* c, const WienerArgs& W) {
  if (W.nb * W.J == 0) return;
  dim3 grid(W.nb, (W.J + kWienerNT - 1) / kWienerNT);
  k_wiener<M, kWienerNT, FROM_X, NOISE><<<grid, kWienerNT, 0, c->stream>>>(W);
  c->launched();
}

// Objective of the current device state -> host double (synchronizes).
template <int M>
double objective(rcscm_gpu_ctx* c, int64_t nb, int64_t J, const rcscm_hyper& h) {
  if (nb * J == 0) return 0.0;
  constexpr int NT = 128;
  dim3 grid(nb, (J + NT - 1) / NT);
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
  const int64_t np = static_cast<int64_t>(grid.x) * grid.y;
  O.partial = c->partial.get<double>(np);
  O.err = c->err.as<unsigned long long>();
  k_objective<M, NT><<<grid, NT, 0, c->stream>>>(O);
  c->launched();
  double* out = c->obj.get<double>(1);
  k_sum_partials<<<1, 1024, 0, c->stream>>>(O.partial, np, out);
  c->launched();
  double v = 0.0;
  d2h(c, &v, out, sizeof(double));
  check_err(c, J);
  return v;
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
    double* tmp = c->tmp.get<double>(S);
    double* tmp2 = c->tmp2.get<double>(S);
    h2d(c, tmp, p->r_h, S * sizeof(double));
    h2d(c, tmp2, p->r_u, S * sizeof(double));
    to_bt<double>(c, tmp, c->rh.as<double>(), 1, I, J);
    to_bt<double>(c, tmp2, c->ru.as<double>(), 1, I, J);
    h2d(c, c->lam.p, p->lambda, I * sizeof(double));
  }
}

void download_params(rcscm_gpu_ctx* c, int64_t I, int64_t J, rcscm_params* out) {
  const size_t S = static_cast<size_t>(I * J);
  double* t1 = c->tmp.get<double>(S);
  double* t2 = c->tmp2.get<double>(S);
  to_ij<double>(c, c->rh.as<double>(), t1, 1, I, J);
  to_ij<double>(c, c->ru.as<double>(), t2, 1, I, J);
  d2h(c, out->r_h, t1, S * sizeof(double));
  d2h(c, out->r_u, t2, S * sizeof(double));
  d2h(c, out->lambda, c->lam.p, I * sizeof(double));
}

void validate_opts(const rcscm_solver_opts* opt, const char* who) {
  if (!opt) fail(RCSCM_INVALID_INPUT, std::string(who) + ": options must not be NULL");
  if (opt->iters < 0) fail(RCSCM_INVALID_INPUT, std::string(who) + ": iters must be >= 0");
}

// Shared driver of run_naive / run_algorithm2 (solver_naive.hpp:412-450,
// solver_accel.hpp:183-240).
void run_solver(rcscm_gpu_ctx* c, bool accel, const rcscm_inputs* in, const rcscm_params* p0,
                const rcscm_hyper* hyper, const double* X, const rcscm_solver_opts* opt, rcscm_params* out,
                rcscm_result* extra) {
  const char* who = accel ? "run_accelerated" : "run_naive";
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
  dispatch_m(M, [&](auto mm) {
    constexpr int MM = decltype(mm)::value;
    upload_model(c, in, p0, X, !accel || opt->compute_objective, accel);
    reset_err(c);
    if (accel) launch_slots<MM>(c, problem(c, 1, I, J, M), false, true, opt->eps_var);
    const bool traj = extra && opt->record_trajectory && (extra->traj_r_h || extra->traj_r_u || extra->traj_lambda);
    const size_t S = static_cast<size_t>(I * J);
    double* trh = traj ? c->traj_rh.get<double>(S * std::max(iters, 1)) : nullptr;
    double* tru = traj ? c->traj_ru.get<double>(S * std::max(iters, 1)) : nullptr;
    double* trl = traj ? c->traj_lam.get<double>(I * std::max(iters, 1)) : nullptr;
    std::vector<double> objv, secs;
    int iters_run = 0;
    auto launch = [&](int first, int count) {
      if (accel) {
        AccelArgs A = accel_args(c, I, J, M, count, *hyper, opt->eps_var, opt->gamma_fault);
        if (traj) {
          A.traj_r_h = trh + static_cast<size_t>(first) * S;
          A.traj_r_u = tru + static_cast<size_t>(first) * S;
          A.traj_lambda = trl + static_cast<size_t>(first) * I;
        }
        launch_accel(c, A);
      } else {
        NaiveArgs N = naive_args(c, I, J, count, *hyper, opt->eps_var);
        if (traj) {
          N.traj_r_h = trh + static_cast<size_t>(first) * S;
          N.traj_r_u = tru + static_cast<size_t>(first) * S;
          N.traj_lambda = trl + static_cast<size_t>(first) * I;
        }
        launch_naive<MM>(c, N);
      }
    };
    if (!opt->compute_objective) {
      CK(cudaEventRecord(c->ev0, c->stream));
      launch(0, iters);
      CK(cudaEventRecord(c->ev1, c->stream));
      iters_run = iters;
      check_err(c, J);
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
      secs.assign(iters, iters ? (ms * 1e-3) / iters : 0.0);
    } else {
      objv.push_back(objective<MM>(c, I, J, *hyper));
      for (int it = 0; it < iters; ++it) {
        CK(cudaEventRecord(c->ev0, c->stream));
        launch(it, 1);
        CK(cudaEventRecord(c->ev1, c->stream));
        ++iters_run;
        objv.push_back(objective<MM>(c, I, J, *hyper));  // synchronizes + checks errors
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
        secs.push_back(ms * 1e-3);
        const double prev = objv[objv.size() - 2], cur = objv.back();
        if (opt->rel_obj_tol > 0.0 && std::abs(cur - prev) <= opt->rel_obj_tol * std::abs(prev)) break;
      }
    }
    download_params(c, I, J, out);
    if (traj && iters_run > 0) {
      double* th = c->tmp.get<double>(S * iters_run);
      if (extra->traj_r_h) {
        to_ij<double>(c, trh, th, iters_run, I, J);
        d2h(c, extra->traj_r_h, th, S * iters_run * sizeof(double));
      }
      if (extra->traj_r_u) {
        to_ij<double>(c, tru, th, iters_run, I, J);
        d2h(c, extra->traj_r_u, th, S * iters_run * sizeof(double));
      }
      d2h(c, extra->traj_lambda, trl, static_cast<size_t>(I) * iters_run * sizeof(double));
    }
    sync(c);
    if (extra) {
      if (extra->objective)
        std::memcpy(extra->objective, objv.data(), objv.size() * sizeof(double));
      if (extra->n_objective) *extra->n_objective = static_cast<int>(objv.size());
      if (extra->iter_seconds) std::memcpy(extra->iter_seconds, secs.data(), secs.size() * sizeof(double));
      if (extra->n_iters) *extra->n_iters = iters_run;
    }
  });
}

}  // namespace

// =============================================================================
// C ABI
// =============================================================================
extern "C" {

const char* rcscm_gpu_last_error(void) { return g_last_error.c_str(); }

int rcscm_gpu_create(const rcscm_gpu_config* cfg, rcscm_gpu_ctx** out) {
  return guarded([&] {
    if (!out) fail(RCSCM_INVALID_INPUT, "out must not be NULL");
    *out = nullptr;
    rcscm_gpu_config d{0, RCSCM_C128, nullptr};
    if (cfg) d = *cfg;
    if (d.precision != RCSCM_C128)
      fail(RCSCM_UNSUPPORTED, "precision: only RCSCM_C128 is implemented in this build");
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    if (d.device < 0 || d.device >= n) fail(RCSCM_INVALID_INPUT, "device ordinal out of range");
    CK(cudaSetDevice(d.device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, d.device));
    if (prop.major != 10)
      fail(RCSCM_UNSUPPORTED, std::string("this build targets sm_100a (B200); device is ") + prop.name);
    auto* c = new rcscm_gpu_ctx();
    c->device = d.device;
    c->precision = d.precision;
    if (d.stream) {
      c->stream = static_cast<cudaStream_t>(d.stream);
    } else {
      CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    CK(cudaEventCreate(&c->ev0));
    CK(cudaEventCreate(&c->ev1));
    *out = c;
  });
}

void rcscm_gpu_destroy(rcscm_gpu_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (DBuf* b : {&c->X, &c->W, &c->A, &c->T, &c->V, &c->a, &c->b, &c->Rp, &c->Rpp, &c->power, &c->sab, &c->taa,
                  &c->sbx, &c->tax, &c->txx, &c->rh, &c->ru, &c->lam, &c->rh0, &c->ru0, &c->lam0, &c->tmp, &c->tmp2,
                  &c->traj_rh, &c->traj_ru, &c->traj_lam, &c->scratch, &c->dry, &c->image, &c->noise,
                  &c->partial, &c->obj, &c->err})
    b->release();
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
}

int64_t rcscm_gpu_launch_count(const rcscm_gpu_ctx* c) { return c ? c->launches : 0; }

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
    dispatch_m(M, [&](auto mm) {
      constexpr int MM = decltype(mm)::value;
      alloc_problem(c, I, J, M);
      c->W.get<double2>(I * M * M);
      c->A.get<double2>(I * M * M);
      h2d(c, c->X.p, X, static_cast<size_t>(I * J * M) * sizeof(double2));
      h2d(c, c->W.p, W, I * M * M * sizeof(double2));
      h2d(c, c->A.p, A, I * M * M * sizeof(double2));
      reset_err(c);
      c->sn_h = n_h;
      DevProblem P = problem(c, 1, I, J, M);
      launch_setup<MM>(c, P, rank_tol, 1e-12);
      check_err(c, J);
      d2h(c, a, c->a.p, I * M * sizeof(double2));
      d2h(c, b, c->b.p, I * M * sizeof(double2));
      d2h(c, Rp, c->Rp.p, I * M * M * sizeof(double2));
      d2h(c, Rpp, c->Rpp.p, I * M * M * sizeof(double2));
      sync(c);
    });
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
    dispatch_m(M, [&](auto mm) {
      constexpr int MM = decltype(mm)::value;
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
      launch_slots<MM>(c, P, true, false, 1e-12);
      k_setup_bin<MM, 1><<<(I + 63) / 64, 64, 0, c->stream>>>(P, 1e-10, 1e-12);
      c->launched();
      check_err(c, J);
      download_params(c, I, J, out);
      sync(c);
    });
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
    dispatch_m(in->mics, [&](auto mm) {
      constexpr int MM = decltype(mm)::value;
      upload_model(c, in, p, X, true, false);
      reset_err(c);
      *out = objective<MM>(c, I, J, *hyper);
    });
  });
}

int rcscm_gpu_run_naive(rcscm_gpu_ctx* c, const rcscm_inputs* in, const rcscm_params* params0,
                        const rcscm_hyper* hyper, const double* X, const rcscm_solver_opts* opt,
                        rcscm_params* out, rcscm_result* extra) {
  return guarded([&] {
    if (!c) fail(RCSCM_INVALID_INPUT, "ctx must not be NULL");
    run_solver(c, false, in, params0, hyper, X, opt, out, extra);
  });
}

int rcscm_gpu_run_algorithm2(rcscm_gpu_ctx* c, const rcscm_inputs* in, const rcscm_params* params0,
                             const rcscm_hyper* hyper, const double* X, const rcscm_solver_opts* opt,
                             rcscm_params* out, rcscm_result* extra) {
  return guarded([&] {
    if (!c) fail(RCSCM_INVALID_INPUT, "ctx must not be NULL");
    run_solver(c, true, in, params0, hyper, X, opt, out, extra);
  });
}

static void extract_impl(rcscm_gpu_ctx* c, const rcscm_inputs* in, const rcscm_params* p, const double* X,
                         double* image, double* dry, double* noise) {
  if (!c || !p) fail(RCSCM_INVALID_INPUT, "extract: NULL argument");
  validate_inputs(in, false, true);
  const int64_t I = in->num_bins, J = in->frames;
  const int M = in->mics;
  if (I == 0) return;
  dispatch_m(M, [&](auto mm) {
    constexpr int MM = decltype(mm)::value;
    upload_model(c, in, p, X, false, true);
    const size_t S = static_cast<size_t>(I * J);
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
    if (noise) {
      Wa.noise = c->noise.get<double2>(S * M);
      launch_wiener<MM, true, true>(c, Wa);
    } else {
      launch_wiener<MM, true, false>(c, Wa);
    }
    if (dry) {
      double2* t = reinterpret_cast<double2*>(c->tmp.get<double2>(S));
      to_ij<double2>(c, Wa.dry, t, 1, I, J);
      d2h(c, dry, t, S * sizeof(double2));
    }
    if (image) d2h(c, image, Wa.image, S * M * sizeof(double2));
    if (noise) d2h(c, noise, Wa.noise, S * M * sizeof(double2));
    sync(c);
  });
}

int rcscm_gpu_extract_target(rcscm_gpu_ctx* c, const rcscm_inputs* in, const rcscm_params* p, const double* X,
                             double* image, double* dry) {
  return guarded([&] { extract_impl(c, in, p, X, image, dry, nullptr); });
}

int rcscm_gpu_extract_noise(rcscm_gpu_ctx* c, const rcscm_inputs* in, const rcscm_params* p, const double* X,
                            double* noise) {
  return guarded([&] {
    if (!noise) fail(RCSCM_INVALID_INPUT, "extract_noise: noise must not be NULL");
    extract_impl(c, in, p, X, nullptr, nullptr, noise);
  });
}

// ---- session ------------------------------------------------------------------
int rcscm_gpu_session_load(rcscm_gpu_ctx* c, int64_t B, int64_t I, int64_t J, int M, int K, int n_h,
                           const double* X, const double* W, const double* A, const double* T, const double* V) {
  return guarded([&] {
    if (!c) fail(RCSCM_INVALID_INPUT, "ctx must not be NULL");
    if (B < 1 || I < 1 || J < 1 || M < 1 || K < 0) fail(RCSCM_INVALID_INPUT, "session_load: bad shape");
    if (n_h < 0 || n_h >= M) fail(RCSCM_INVALID_INPUT, "session_load: target index out of range");
    dispatch_m(M, [&](auto) {});
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
    h2d(c, c->X.p, X, S * M * sizeof(double2));
    h2d(c, c->W.p, W, nb * M * M * sizeof(double2));
    h2d(c, c->A.p, A, nb * M * M * sizeof(double2));
    h2d(c, c->T.p, T, B * I * K * sizeof(double));
    h2d(c, c->V.p, V, B * K * J * sizeof(double));
    c->sB = B;
    c->sI = I;
    c->sJ = J;
    c->sM = M;
    c->sK = K;
    c->sn_h = n_h;
    c->s_loaded = true;
    c->s_setup = false;
    c->s_pre = false;
    reset_err(c);
    sync(c);
  });
}

int rcscm_gpu_session_run(rcscm_gpu_ctx* c, int stages, int iters, const rcscm_hyper* hyper, double eps_var) {
  return guarded([&] {
    if (!c || !c->s_loaded) fail(RCSCM_INVALID_INPUT, "session_run: no session loaded");
    if (iters < 0) fail(RCSCM_INVALID_INPUT, "session_run: iters must be >= 0");
    const rcscm_hyper h = hyper ? *hyper : rcscm_hyper{1.1, 1e-16};
    const int64_t nb = c->sB * c->sI, J = c->sJ;
    const int M = c->sM;
    const size_t S = static_cast<size_t>(nb * J);
    dispatch_m(M, [&](auto mm) {
      constexpr int MM = decltype(mm)::value;
      DevProblem P = problem(c, c->sB, c->sI, J, M);
      bool pre_done = false;
      if (stages & RCSCM_STAGE_SETUP) {
        launch_setup<MM>(c, P, 1e-10, eps_var);
        const bool pre = (stages & RCSCM_STAGE_PRECOMPUTE) != 0;
        launch_slots<MM>(c, P, true, pre, eps_var);
        pre_done = pre;
        CK(cudaMemcpyAsync(c->rh0.p, c->rh.p, S * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaMemcpyAsync(c->ru0.p, c->ru.p, S * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaMemcpyAsync(c->lam0.p, c->lam.p, nb * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
        c->s_setup = true;
        if (pre) c->s_pre = true;
      }
      if (!c->s_setup) fail(RCSCM_INVALID_INPUT, "session_run: run RCSCM_STAGE_SETUP first");
      if (stages & RCSCM_STAGE_RESET) {
        CK(cudaMemcpyAsync(c->rh.p, c->rh0.p, S * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaMemcpyAsync(c->ru.p, c->ru0.p, S * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaMemcpyAsync(c->lam.p, c->lam0.p, nb * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
      }
      if ((stages & RCSCM_STAGE_PRECOMPUTE) && !pre_done) {
        launch_slots<MM>(c, P, false, true, eps_var);
        c->s_pre = true;
      }
      if (stages & RCSCM_STAGE_ACCEL) {
        if (!c->s_pre) fail(RCSCM_INVALID_INPUT, "session_run: ACCEL needs PRECOMPUTE");
        launch_accel(c, accel_args(c, nb, J, M, iters, h, eps_var, 0.0));
      }
      if (stages & RCSCM_STAGE_NAIVE) launch_naive<MM>(c, naive_args(c, nb, J, iters, h, eps_var));
      if (stages & RCSCM_STAGE_WIENER) {
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
        launch_wiener<MM, false, false>(c, Wa);
      }
    });
  });
}

int rcscm_gpu_session_fetch(rcscm_gpu_ctx* c, double* r_h, double* r_u, double* lambda, double* dry,
                            double* image, int do_sync) {
  return guarded([&] {
    if (!c || !c->s_loaded) fail(RCSCM_INVALID_INPUT, "session_fetch: no session loaded");
    const int64_t nb = c->sB * c->sI, J = c->sJ;
    const size_t S = static_cast<size_t>(nb * J);
    d2h(c, r_h, c->rh.p, S * sizeof(double));
    d2h(c, r_u, c->ru.p, S * sizeof(double));
    d2h(c, lambda, c->lam.p, nb * sizeof(double));
    d2h(c, dry, c->dry.p, S * sizeof(double2));
    d2h(c, image, c->image.p, S * c->sM * sizeof(double2));
    if (do_sync) sync(c);
  });
}

int rcscm_gpu_session_check(rcscm_gpu_ctx* c) {
  return guarded([&] {
    if (!c || !c->s_loaded) fail(RCSCM_INVALID_INPUT, "session_check: no session loaded");
    check_err(c, c->sJ);
  });
}

int rcscm_gpu_probe_fp64(rcscm_gpu_ctx* c, double* tflops, double* ms) {
  return guarded([&] {
    if (!c || !tflops) fail(RCSCM_INVALID_INPUT, "probe_fp64: NULL argument");
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
    constexpr int NACC = 8, NT = 256;
    const int blocks = sms * 8, iters = 20000;
    double* out = c->obj.get<double>(1);
    k_fp64_probe<NACC><<<blocks, NT, 0, c->stream>>>(1.0, iters / 10, out);  // warm-up
    c->launched();
    CK(cudaEventRecord(c->ev0, c->stream));
    k_fp64_probe<NACC><<<blocks, NT, 0, c->stream>>>(1.0, iters, out);
    c->launched();
    CK(cudaEventRecord(c->ev1, c->stream));
    CK(cudaEventSynchronize(c->ev1));
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, c->ev0, c->ev1));
    const double flops = 2.0 * NACC * static_cast<double>(iters) * blocks * NT;
    *tflops = flops / (t * 1e-3) / 1e12;
    if (ms) *ms = t;
  });
}

}  // extern "C"
