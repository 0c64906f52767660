// rcscm_oracle.cpp -- CPU ORACLE for the rank-constrained SCM hot path.
//
// TEST INFRASTRUCTURE ONLY. This file restates, in plain C++17 with
// std::complex<double>, the reference algorithm of
//   /root/reference/proj/include/rcscm/linalg.hpp        (eig, pinv, null vector)
//   /root/reference/proj/include/rcscm/model.hpp         (build_noise_scm, init_params, map_objective)
//   /root/reference/proj/include/rcscm/ilrma.hpp         (sphere, run_ilrma, ilrma_objective,
//                                                         scale_fixed_noise_image; Eigen::FullPivLU
//                                                         restated with its pivot and rank rules)
//   /root/reference/proj/include/rcscm/solver_accel.hpp  (Algorithms 1 and 2)
//   /root/reference/proj/include/rcscm/solver_naive.hpp  (naive EM)
//   /root/reference/proj/include/rcscm/wiener.hpp        (MWF extraction)
//   /root/reference/proj/include/rcscm/verify.hpp        (seeded instances, parity metric)
// The reference itself cannot be compiled here (it needs Eigen 3, absent from the
// image), so Eigen's SelfAdjointEigenSolver is replaced by a cyclic complex Jacobi
// solver and Eigen::LLT by a hand complex Cholesky; per-slot formulas, evaluation
// order, flooring and snapshot semantics follow the reference line by line.
//
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
// reference legs) may load this library, and only as the checker. The product
// path (paper_1908_01964_b200/) never links or calls it.

#include "rcscm_oracle.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace oracle {

using cplx = std::complex<double>;
using Index = int64_t;

constexpr double kEpsVar = 1e-12;          // types.hpp:55
constexpr double kDefaultRankTol = 1e-10;  // linalg.hpp:12

// types.hpp:20-30
struct InvalidInputError : std::invalid_argument {
  explicit InvalidInputError(const std::string& w) : std::invalid_argument(w) {}
};
struct NumericalError : std::runtime_error {
  explicit NumericalError(const std::string& w) : std::runtime_error(w) {}
};

// Dense column-major complex matrix (stand-in for Eigen::MatrixXcd).
struct CMat {
  int rows = 0, cols = 0;
  std::vector<cplx> d;
  CMat() = default;
  CMat(int r, int c) : rows(r), cols(c), d(static_cast<size_t>(r) * c, cplx(0, 0)) {}
  cplx& operator()(int r, int c) { return d[r + static_cast<size_t>(c) * rows]; }
  const cplx& operator()(int r, int c) const { return d[r + static_cast<size_t>(c) * rows]; }
  static CMat identity(int n) {
    CMat m(n, n);
    for (int k = 0; k < n; ++k) m(k, k) = 1.0;
    return m;
  }
};
using CVec = std::vector<cplx>;

static CMat load_mat(const double* p, int M) {
  CMat m(M, M);
  std::memcpy(m.d.data(), p, sizeof(cplx) * M * M);
  return m;
}
static void store_mat(const CMat& m, double* p) {
  std::memcpy(p, m.d.data(), sizeof(cplx) * m.d.size());
}
static CVec load_vec(const double* p, int M) {
  CVec v(M);
  std::memcpy(v.data(), p, sizeof(cplx) * M);
  return v;
}
static const cplx* C(const double* p) { return reinterpret_cast<const cplx*>(p); }
static cplx* C(double* p) { return reinterpret_cast<cplx*>(p); }

static double frob(const CMat& m) {
  double s = 0;
  for (const cplx& z : m.d) s += std::norm(z);
  return std::sqrt(s);
}

// Static chunked parallel-for with first-exception propagation, as
// parallel.hpp:50-80 (threads spawned per call, deterministic per index).
static void parallel_for_chunks(Index begin, Index end, int threads,
                                const std::function<void(Index, Index)>& body) {
  const Index n = end - begin;
  if (n <= 0) return;
  if (threads <= 1 || n == 1) {
    body(begin, end);
    return;
  }
  const int workers = static_cast<int>(std::min<Index>(threads, n));
  std::exception_ptr first;
  std::mutex mu;
  std::vector<std::thread> pool;
  const Index chunk = (n + workers - 1) / workers;
  for (int w = 0; w < workers; ++w) {
    const Index lo = begin + w * chunk, hi = std::min(end, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back([lo, hi, &body, &first, &mu] {
      try {
        body(lo, hi);
      } catch (...) {
        std::lock_guard<std::mutex> g(mu);
        if (!first) first = std::current_exception();
      }
    });
  }
  for (auto& t : pool) t.join();
  if (first) std::rethrow_exception(first);
}

// ---------------------------------------------------------------------------
// linalg.hpp
// ---------------------------------------------------------------------------

// linalg.hpp:14-17
static bool is_hermitian(const CMat& H, double rel_tol = 1e-12) {
  double diff = 0;
  for (int c = 0; c < H.cols; ++c)
    for (int r = 0; r < H.rows; ++r) diff += std::norm(H(r, c) - std::conj(H(c, r)));
  const double scale = std::max(frob(H), 1.0);
  return std::sqrt(diff) <= rel_tol * scale;
}

struct EigResult {
  std::vector<double> values;  // ascending
  CMat vectors;                // column k pairs with values[k]
};

// linalg.hpp:25-34 hermitian_eig. Eigen's SelfAdjointEigenSolver is replaced
// by cyclic complex Jacobi: each rotation J = diag(1, conj(e)) * [[c, s], [-s, c]]
// on (p, q), with e the phase of H(p, q), zeroes H(p, q); sweeps repeat until no
// off-diagonal entry exceeds 1e-18 * ||H||_F. Eigenvalues are sorted ascending.
static EigResult hermitian_eig(const CMat& H) {
  if (H.rows != H.cols || H.rows < 1)
    throw InvalidInputError("hermitian_eig: matrix must be square and nonempty");
  if (!is_hermitian(H)) throw InvalidInputError("hermitian_eig: input is not Hermitian");
  const int n = H.rows;
  CMat A = H;
  // Work on the exactly-Hermitian part (Eigen reads the lower triangle only).
  for (int c = 0; c < n; ++c) {
    A(c, c) = cplx(std::real(H(c, c)), 0.0);
    for (int r = c + 1; r < n; ++r) {
      A(r, c) = H(r, c);
      A(c, r) = std::conj(H(r, c));
    }
  }
  CMat V = CMat::identity(n);
  const double thresh = 1e-18 * frob(A);
  bool finite = true;
  for (const cplx& z : A.d) finite = finite && std::isfinite(z.real()) && std::isfinite(z.imag());
  if (!finite) throw NumericalError("hermitian_eig: eigensolver failed to converge");
  for (int sweep = 0; sweep < 100; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < n - 1; ++p) {
      for (int q = p + 1; q < n; ++q) {
        const cplx g = A(p, q);
        const double ag = std::abs(g);
        if (!(ag > thresh)) continue;
        rotated = true;
        const double app = std::real(A(p, p)), aqq = std::real(A(q, q));
        const double tau = (aqq - app) / (2.0 * ag);
        const double t = (tau >= 0 ? 1.0 : -1.0) / (std::abs(tau) + std::sqrt(1.0 + tau * tau));
        const double c = 1.0 / std::sqrt(1.0 + t * t);
        const double s = t * c;
        const cplx e = g / ag;
        const cplx eb = std::conj(e);
        for (int k = 0; k < n; ++k) {  // A <- A J
          const cplx akp = A(k, p), akq = A(k, q);
          A(k, p) = c * akp - s * eb * akq;
          A(k, q) = s * akp + c * eb * akq;
        }
        for (int k = 0; k < n; ++k) {  // A <- J^H A
          const cplx apk = A(p, k), aqk = A(q, k);
          A(p, k) = c * apk - s * e * aqk;
          A(q, k) = s * apk + c * e * aqk;
        }
        A(p, q) = A(q, p) = cplx(0, 0);
        A(p, p) = cplx(app - t * ag, 0.0);
        A(q, q) = cplx(aqq + t * ag, 0.0);
        for (int k = 0; k < n; ++k) {  // V <- V J
          const cplx vkp = V(k, p), vkq = V(k, q);
          V(k, p) = c * vkp - s * eb * vkq;
          V(k, q) = s * vkp + c * eb * vkq;
        }
      }
    }
    if (!rotated) break;
  }
  std::vector<int> order(n);
  for (int k = 0; k < n; ++k) order[k] = k;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
    return std::real(A(x, x)) < std::real(A(y, y));
  });
  EigResult out;
  out.values.resize(n);
  out.vectors = CMat(n, n);
  for (int k = 0; k < n; ++k) {
    out.values[k] = std::real(A(order[k], order[k]));
    for (int r = 0; r < n; ++r) out.vectors(r, k) = V(r, order[k]);
  }
  return out;
}

// linalg.hpp:38-53
static CMat pseudo_inverse_psd(const CMat& H, double rank_tol = kDefaultRankTol) {
  const EigResult eig = hermitian_eig(H);
  const int m = H.rows;
  const double lmax = std::max(eig.values[m - 1], 0.0);
  const double cutoff = rank_tol * lmax;
  if (eig.values[0] < -cutoff)
    throw InvalidInputError("pseudo_inverse_psd: matrix is not PSD (eigenvalue " +
                            std::to_string(eig.values[0]) + ")");
  CMat pinv(m, m);
  for (int k = 0; k < m; ++k) {
    if (eig.values[k] > cutoff) {
      const double inv = 1.0 / eig.values[k];
      for (int c = 0; c < m; ++c)
        for (int r = 0; r < m; ++r)
          pinv(r, c) += (inv * eig.vectors(r, k)) * std::conj(eig.vectors(c, k));
    }
  }
  return pinv;
}

// linalg.hpp:58-70
static CVec normalize_phase(const CVec& v) {
  double vmax = 0;
  for (const cplx& z : v) vmax = std::max(vmax, std::abs(z));
  if (vmax == 0.0) return v;
  size_t pivot_idx = 0;
  for (size_t k = 0; k < v.size(); ++k) {
    if (std::abs(v[k]) > 1e-8 * vmax) {
      pivot_idx = k;
      break;
    }
  }
  const cplx pivot = v[pivot_idx];
  const cplx f = std::conj(pivot) / std::abs(pivot);
  CVec out(v.size());
  for (size_t k = 0; k < v.size(); ++k) out[k] = v[k] * f;
  return out;
}

// linalg.hpp:74-86
static CVec null_eigenvector(const CMat& Rp, double rank_tol = kDefaultRankTol) {
  const EigResult eig = hermitian_eig(Rp);
  const int m = Rp.rows;
  const double lmax = std::max(eig.values[m - 1], 0.0);
  const double cutoff = rank_tol * std::max(lmax, 1e-300);
  int near_zero = 0;
  for (int k = 0; k < m; ++k)
    if (eig.values[k] <= cutoff) ++near_zero;
  if (near_zero != 1)
    throw InvalidInputError(
        "null_eigenvector: expected exactly one near-zero eigenvalue, found " +
        std::to_string(near_zero));
  CVec v0(m);
  for (int r = 0; r < m; ++r) v0[r] = eig.vectors(r, 0);
  return normalize_phase(v0);
}

// linalg.hpp:90-101
static CMat sherman_morrison_inverse(const CMat& Rinv, const CVec& a, double c, double d) {
  if (d <= 0.0)
    throw InvalidInputError("sherman_morrison_inverse: noise variance must be > 0");
  const int m = Rinv.rows;
  CVec ra(m, 0.0);
  for (int r = 0; r < m; ++r)
    for (int k = 0; k < m; ++k) ra[r] += Rinv(r, k) * a[k];
  cplx quadc = 0;
  for (int r = 0; r < m; ++r) quadc += std::conj(a[r]) * ra[r];
  const double gain = c / (d + c * std::real(quadc));
  CMat out = Rinv;
  for (int cc = 0; cc < m; ++cc)
    for (int r = 0; r < m; ++r) out(r, cc) -= (gain * ra[r]) * std::conj(ra[cc]);
  for (auto& z : out.d) z *= (1.0 / d);
  return out;
}

// linalg.hpp:105-117
static CMat rank_one_restored_inverse(const CMat& Rpp, const CVec& b, double lambda) {
  if (lambda <= 0.0)
    throw InvalidInputError("rank_one_restored_inverse: lambda must be > 0");
  const int m = Rpp.rows;
  double bn = 0;
  for (const cplx& z : b) bn += std::norm(z);
  if (std::abs(std::sqrt(bn) - 1.0) > 1e-10)
    throw InvalidInputError("rank_one_restored_inverse: b must be unit norm");
  double res = 0;
  for (int r = 0; r < m; ++r) {
    cplx acc = 0;
    for (int k = 0; k < m; ++k) acc += Rpp(r, k) * b[k];
    res += std::norm(acc);
  }
  if (std::sqrt(res) > 1e-8 * std::max(frob(Rpp), 1.0))
    throw InvalidInputError(
        "rank_one_restored_inverse: b is not in the null space of the pseudoinverse");
  CMat out = Rpp;
  for (int c = 0; c < m; ++c)
    for (int r = 0; r < m; ++r) out(r, c) += ((1.0 / lambda) * b[r]) * std::conj(b[c]);
  return out;
}

// Complex Cholesky (Eigen::LLT stand-in, lower triangle read). Returns false
// when a pivot is <= 0, as LLT::info() != Success (Eigen's own test, so a NaN
// pivot is not caught here and surfaces later as a non-finite value).
static bool llt(const CMat& A, CMat* L) {
  const int n = A.rows;
  *L = CMat(n, n);
  for (int k = 0; k < n; ++k) {
    double x = std::real(A(k, k));
    for (int j = 0; j < k; ++j) x -= std::norm((*L)(k, j));
    if (x <= 0.0) return false;  // Eigen LLT test: a NaN pivot passes on
    const double lkk = std::sqrt(x);
    (*L)(k, k) = lkk;
    for (int i = k + 1; i < n; ++i) {
      cplx s = A(i, k);
      for (int j = 0; j < k; ++j) s -= (*L)(i, j) * std::conj((*L)(k, j));
      (*L)(i, k) = s / lkk;
    }
  }
  return true;
}
// Solve L L^H z = rhs in place (rhs columns).
static void llt_solve_inplace(const CMat& L, CMat* B) {
  const int n = L.rows;
  for (int col = 0; col < B->cols; ++col) {
    for (int i = 0; i < n; ++i) {
      cplx s = (*B)(i, col);
      for (int j = 0; j < i; ++j) s -= L(i, j) * (*B)(j, col);
      (*B)(i, col) = s / std::real(L(i, i));
    }
    for (int i = n - 1; i >= 0; --i) {
      cplx s = (*B)(i, col);
      for (int j = i + 1; j < n; ++j) s -= std::conj(L(j, i)) * (*B)(j, col);
      (*B)(i, col) = s / std::real(L(i, i));
    }
  }
}

// ---------------------------------------------------------------------------
// model.hpp
// ---------------------------------------------------------------------------

struct Inputs {  // model.hpp:16-25 RcscmInputs
  Index I = 0;
  int M = 0;
  int n_h = 0;
  std::vector<CVec> a, b;
  std::vector<CMat> Rp, Rpp;
};
struct Params {  // model.hpp:29-33 RcscmParams (r_h/r_u I x J column-major)
  Index I = 0, J = 0;
  std::vector<double> r_h, r_u, lambda;
  double& rh(Index i, Index t) { return r_h[i + t * I]; }
  double& ru(Index i, Index t) { return r_u[i + t * I]; }
  double rh(Index i, Index t) const { return r_h[i + t * I]; }
  double ru(Index i, Index t) const { return r_u[i + t * I]; }
};
struct Spec {  // types.hpp:43-53 Spectrogram, bins[i] = M x J col-major
  Index I = 0, J = 0;
  int M = 0;
  const cplx* x = nullptr;
  const cplx* col(Index i, Index t) const { return x + (i * J + t) * M; }
};
struct Hyper {  // model.hpp:36-39
  double alpha = 1.1, beta = 1e-16;
};

static Inputs make_inputs(Index I, int M, const double* a, const double* Rp,
                          const double* Rpp, const double* b) {
  Inputs in;
  in.I = I;
  in.M = M;
  in.a.resize(I);
  in.b.resize(I);
  in.Rp.resize(I);
  in.Rpp.resize(I);
  for (Index i = 0; i < I; ++i) {
    if (a) in.a[i] = load_vec(a + 2 * i * M, M);
    if (b) in.b[i] = load_vec(b + 2 * i * M, M);
    if (Rp) in.Rp[i] = load_mat(Rp + 2 * i * M * M, M);
    if (Rpp) in.Rpp[i] = load_mat(Rpp + 2 * i * M * M, M);
  }
  return in;
}
static Params make_params(Index I, Index J, const double* r_h, const double* r_u,
                          const double* lam) {
  Params p;
  p.I = I;
  p.J = J;
  p.r_h.assign(r_h, r_h + I * J);
  p.r_u.assign(r_u, r_u + I * J);
  p.lambda.assign(lam, lam + I);
  return p;
}

// model.hpp:58-90 build_noise_scm
static void build_noise_scm(const std::vector<CMat>& W, const std::vector<CMat>& A,
                            const Spec& X, int n_h, double rank_tol, Inputs* in) {
  const Index I = X.I, J = X.J;
  const int m = X.M;
  if (n_h < 0 || n_h >= m) throw InvalidInputError("build_noise_scm: target index out of range");
  in->I = I;
  in->M = m;
  in->n_h = n_h;
  in->a.assign(I, CVec());
  in->b.assign(I, CVec());
  in->Rp.assign(I, CMat());
  in->Rpp.assign(I, CMat());
  for (Index i = 0; i < I; ++i) {
    CVec a(m);
    for (int r = 0; r < m; ++r) a[r] = A[i](r, n_h);
    in->a[i] = a;
    std::vector<double> mean_power(m, 0.0);
    for (int n = 0; n < m; ++n) {
      if (n == n_h) continue;
      double acc = 0;
      for (Index t = 0; t < J; ++t) {
        const cplx* x = X.col(i, t);
        cplx y = 0;
        for (int k = 0; k < m; ++k) y += W[i](n, k) * x[k];
        acc += std::norm(y);
      }
      mean_power[n] = acc / static_cast<double>(J);
    }
    CMat rp(m, m);
    for (int c = 0; c < m; ++c)
      for (int r = 0; r < m; ++r) {
        cplx s = 0;
        for (int n = 0; n < m; ++n) s += (A[i](r, n) * mean_power[n]) * std::conj(A[i](c, n));
        rp(r, c) = s;
      }
    CMat sym(m, m);
    for (int c = 0; c < m; ++c)
      for (int r = 0; r < m; ++r) sym(r, c) = (rp(r, c) + std::conj(rp(c, r))) / 2.0;
    in->Rp[i] = sym;
    try {
      in->b[i] = null_eigenvector(sym, rank_tol);
      in->Rpp[i] = pseudo_inverse_psd(sym, rank_tol);
    } catch (const InvalidInputError& e) {
      throw InvalidInputError("build_noise_scm: frequency bin " + std::to_string(i) + ": " +
                              e.what());
    }
  }
}

// ilrma.hpp:78-83 scale_fixed_noise_image
static CVec scale_fixed_noise_image(const CMat& W, const CMat& A, const cplx* x, int n_h) {
  const int m = W.rows;
  CVec y(m, 0.0);
  for (int r = 0; r < m; ++r)
    for (int k = 0; k < m; ++k) y[r] += W(r, k) * x[k];
  y[n_h] = cplx(0.0, 0.0);
  CVec out(m, 0.0);
  for (int r = 0; r < m; ++r)
    for (int k = 0; k < m; ++k) out[r] += A(r, k) * y[k];
  return out;
}

// model.hpp:95-124 init_params
static void init_params(const Inputs& in, const double* T, const double* V, int K,
                        const std::vector<CMat>& W, const std::vector<CMat>& A,
                        const Spec& X, Params* p) {
  const Index I = X.I, J = X.J;
  const int m = X.M;
  p->I = I;
  p->J = J;
  p->r_h.assign(I * J, 0.0);
  p->r_u.assign(I * J, 0.0);
  p->lambda.assign(I, 0.0);
  for (Index t = 0; t < J; ++t)
    for (Index i = 0; i < I; ++i) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += T[i + k * I] * V[k + t * K];
      p->rh(i, t) = std::max(s, kEpsVar);
    }
  for (Index i = 0; i < I; ++i) {
    for (Index t = 0; t < J; ++t) {
      const CVec yh = scale_fixed_noise_image(W[i], A[i], X.col(i, t), in.n_h);
      cplx q = 0;
      for (int r = 0; r < m; ++r) {
        cplx acc = 0;
        for (int k = 0; k < m; ++k) acc += in.Rpp[i](r, k) * yh[k];
        q += std::conj(yh[r]) * acc;
      }
      p->ru(i, t) = std::max(std::real(q) / m, kEpsVar);
    }
    const EigResult eig = hermitian_eig(in.Rp[i]);
    const double cutoff = kDefaultRankTol * std::max(eig.values[m - 1], 0.0);
    double lmin = eig.values[m - 1];
    for (int k = 0; k < m; ++k) {
      if (eig.values[k] > cutoff) {
        lmin = eig.values[k];
        break;
      }
    }
    p->lambda[i] = std::max(lmin, kEpsVar);
  }
}

// model.hpp:129-157 map_objective
static double map_objective(const Inputs& in, const Params& p, const Hyper& hyper,
                            const Spec& X) {
  const Index I = X.I, J = X.J;
  const int m = X.M;
  double obj = 0.0;
  for (Index i = 0; i < I; ++i) {
    CMat Ru = in.Rp[i];
    for (int c = 0; c < m; ++c)
      for (int r = 0; r < m; ++r)
        Ru(r, c) += (p.lambda[i] * in.b[i][r]) * std::conj(in.b[i][c]);
    for (Index t = 0; t < J; ++t) {
      CMat Rx(m, m);
      const double rh = p.rh(i, t), ru = p.ru(i, t);
      for (int c = 0; c < m; ++c)
        for (int r = 0; r < m; ++r)
          Rx(r, c) = (rh * in.a[i][r]) * std::conj(in.a[i][c]) + ru * Ru(r, c);
      CMat L;
      if (!llt(Rx, &L))
        throw NumericalError("map_objective: R^(x) not PD at bin " + std::to_string(i) +
                             ", frame " + std::to_string(t));
      double logdet = m * std::log(M_PI);
      for (int k = 0; k < m; ++k) logdet += 2.0 * std::log(std::real(L(k, k)));
      CMat z(m, 1);
      const cplx* x = X.col(i, t);
      for (int k = 0; k < m; ++k) z(k, 0) = x[k];
      llt_solve_inplace(L, &z);
      cplx q = 0;
      for (int k = 0; k < m; ++k) q += std::conj(x[k]) * z(k, 0);
      obj += -logdet - std::real(q) - (hyper.alpha + 1.0) * std::log(rh) - hyper.beta / rh;
      if (!std::isfinite(obj))
        throw NumericalError("map_objective: non-finite at bin " + std::to_string(i) +
                             ", frame " + std::to_string(t));
    }
  }
  return obj;
}

// ---------------------------------------------------------------------------
// solver_accel.hpp
// ---------------------------------------------------------------------------

struct Scratch {  // solver_accel.hpp:18-30 (I x J arrays column-major)
  Index I = 0, J = 0;
  std::vector<cplx> sigma_ab, sigma_bx, tau_ax, rho_ax, trho_ax;
  std::vector<double> tau_aa, tau_xx, rho_aa, trho_aa, rho_xx, gamma;
};

// solver_accel.hpp:33-43
static void precompute_sigma(const Inputs& in, const Spec& X, Scratch* s) {
  const Index I = X.I, J = X.J;
  const int m = X.M;
  s->I = I;
  s->J = J;
  s->sigma_ab.assign(I, 0.0);
  s->sigma_bx.assign(I * J, 0.0);
  for (Index i = 0; i < I; ++i) {
    cplx ab = 0;
    for (int k = 0; k < m; ++k) ab += std::conj(in.a[i][k]) * in.b[i][k];
    s->sigma_ab[i] = ab;
    for (Index t = 0; t < J; ++t) {
      const cplx* x = X.col(i, t);
      cplx v = 0;
      for (int k = 0; k < m; ++k) v += std::conj(in.b[i][k]) * x[k];
      s->sigma_bx[i + t * I] = v;
    }
  }
}

// solver_accel.hpp:47-64
static void precompute_tau(const Inputs& in, const Spec& X, Scratch* s) {
  const Index I = X.I, J = X.J;
  const int m = X.M;
  s->tau_aa.assign(I, 0.0);
  s->tau_ax.assign(I * J, 0.0);
  s->tau_xx.assign(I * J, 0.0);
  for (Index i = 0; i < I; ++i) {
    const CMat& P = in.Rpp[i];
    CVec pa(m, 0.0);
    for (int r = 0; r < m; ++r)
      for (int k = 0; k < m; ++k) pa[r] += P(r, k) * in.a[i][k];
    cplx aa = 0;
    for (int k = 0; k < m; ++k) aa += std::conj(in.a[i][k]) * pa[k];
    s->tau_aa[i] = std::max(std::real(aa), 0.0);
    for (Index t = 0; t < J; ++t) {
      const cplx* x = X.col(i, t);
      cplx ax = 0;
      for (int k = 0; k < m; ++k) ax += std::conj(pa[k]) * x[k];
      s->tau_ax[i + t * I] = ax;
      cplx xx = 0;
      for (int r = 0; r < m; ++r) {
        cplx acc = 0;
        for (int k = 0; k < m; ++k) acc += P(r, k) * x[k];
        xx += std::conj(x[r]) * acc;
      }
      s->tau_xx[i + t * I] = std::max(std::real(xx), 0.0);
    }
  }
}

// solver_accel.hpp:67-76
static void compute_gamma(const Params& tilde, const std::vector<double>& trho_aa,
                          Scratch* s) {
  const Index I = tilde.I, J = tilde.J;
  s->gamma.assign(I * J, 0.0);
  for (Index i = 0; i < I; ++i)
    for (Index t = 0; t < J; ++t)
      s->gamma[i + t * I] = tilde.rh(i, t) / (tilde.ru(i, t) + tilde.rh(i, t) * trho_aa[i]);
}

// solver_accel.hpp:80-109
static void rho_first_stage(const Inputs& in, const Spec& X, const std::vector<double>& lambda,
                            std::vector<double>* rho_aa, std::vector<cplx>* rho_ax,
                            std::vector<double>* rho_xx, int threads) {
  const Index I = X.I, J = X.J;
  const int m = X.M;
  rho_aa->assign(I, 0.0);
  rho_ax->assign(I * J, 0.0);
  if (rho_xx) rho_xx->assign(I * J, 0.0);
  parallel_for_chunks(0, I, threads, [&](Index lo, Index hi) {
    for (Index i = lo; i < hi; ++i) {
      if (lambda[i] <= 0.0)
        throw NumericalError("rho_first_stage: nonpositive lambda at bin " + std::to_string(i));
      CMat Ru = in.Rp[i];
      for (int c = 0; c < m; ++c)
        for (int r = 0; r < m; ++r)
          Ru(r, c) += (lambda[i] * in.b[i][r]) * std::conj(in.b[i][c]);
      CMat L;
      if (!llt(Ru, &L))
        throw NumericalError("rho_first_stage: singular R^(u) at bin " + std::to_string(i));
      CMat Rinv = CMat::identity(m);
      llt_solve_inplace(L, &Rinv);
      CVec ria(m, 0.0);
      for (int r = 0; r < m; ++r)
        for (int k = 0; k < m; ++k) ria[r] += Rinv(r, k) * in.a[i][k];
      cplx aa = 0;
      for (int k = 0; k < m; ++k) aa += std::conj(in.a[i][k]) * ria[k];
      (*rho_aa)[i] = std::real(aa);
      for (Index t = 0; t < J; ++t) {
        const cplx* x = X.col(i, t);
        cplx ax = 0;
        for (int k = 0; k < m; ++k) ax += std::conj(ria[k]) * x[k];
        (*rho_ax)[i + t * I] = ax;
        if (rho_xx) {
          cplx xx = 0;
          for (int r = 0; r < m; ++r) {
            cplx acc = 0;
            for (int k = 0; k < m; ++k) acc += Rinv(r, k) * x[k];
            xx += std::conj(x[r]) * acc;
          }
          (*rho_xx)[i + t * I] = std::real(xx);
        }
      }
    }
  });
}

// solver_accel.hpp:113-129
static void rho_second_stage(const Scratch& s, const std::vector<double>& lambda,
                             std::vector<double>* rho_aa, std::vector<cplx>* rho_ax,
                             std::vector<double>* rho_xx) {
  const Index I = s.I, J = s.J;
  rho_aa->assign(I, 0.0);
  rho_ax->assign(I * J, 0.0);
  if (rho_xx) rho_xx->assign(I * J, 0.0);
  for (Index i = 0; i < I; ++i) {
    const double inv_lam = 1.0 / lambda[i];
    (*rho_aa)[i] = s.tau_aa[i] + std::norm(s.sigma_ab[i]) * inv_lam;
    for (Index t = 0; t < J; ++t) {
      (*rho_ax)[i + t * I] = s.tau_ax[i + t * I] + s.sigma_ab[i] * s.sigma_bx[i + t * I] * inv_lam;
      if (rho_xx) (*rho_xx)[i + t * I] = s.tau_xx[i + t * I] + std::norm(s.sigma_bx[i + t * I]) * inv_lam;
    }
  }
}

// solver_accel.hpp:134-141
static void update_rh(const Scratch& s, const Params& tilde, const Hyper& h, double eps,
                      std::vector<double>* r_h) {
  const Index n = tilde.I * tilde.J;
  r_h->assign(n, 0.0);
  for (Index k = 0; k < n; ++k) {
    const double g = s.gamma[k];
    const double v = (g * (tilde.r_u[k] + g * std::norm(s.trho_ax[k])) + h.beta) / (h.alpha + 2.0);
    (*r_h)[k] = std::max(v, eps);
  }
}

// solver_accel.hpp:143-158
static void update_lambda(const Scratch& s, const Params& tilde, double eps,
                          std::vector<double>* lambda) {
  const Index I = tilde.I, J = tilde.J;
  lambda->assign(I, 0.0);
  for (Index i = 0; i < I; ++i) {
    const double ab2 = std::norm(s.sigma_ab[i]);
    double acc = 0.0;
    for (Index t = 0; t < J; ++t) {
      const Index k = i + t * I;
      const cplx resid = s.sigma_bx[k] - s.gamma[k] * std::conj(s.sigma_ab[i]) * s.trho_ax[k];
      acc += s.gamma[k] * ab2 + std::norm(resid) / tilde.r_u[k];
    }
    (*lambda)[i] = std::max(acc / static_cast<double>(J), eps);
  }
}

// solver_accel.hpp:160-176
static void update_ru(const Scratch& s, const Params& tilde, int mics, double eps,
                      std::vector<double>* r_u) {
  const Index I = tilde.I, J = tilde.J;
  r_u->assign(I * J, 0.0);
  for (Index i = 0; i < I; ++i) {
    for (Index t = 0; t < J; ++t) {
      const Index k = i + t * I;
      const double g = s.gamma[k];
      const double val = (g * s.rho_aa[i] * (tilde.r_u[k] + g * std::norm(s.trho_ax[k])) +
                          s.rho_xx[k] - 2.0 * g * std::real(s.trho_ax[k] * std::conj(s.rho_ax[k]))) /
                         static_cast<double>(mics);
      (*r_u)[k] = std::max(val, eps);
    }
  }
}

struct Options {  // solver_naive.hpp:14-22 SolverOptions
  int iters = 200;
  bool compute_objective = false;
  bool record_trajectory = false;
  double rel_obj_tol = 0.0;
  int threads = 1;
  double eps_var = kEpsVar;
  double gamma_fault = 0.0;
};
struct Result {  // solver_naive.hpp:24-29 SolverResult
  Params params;
  std::vector<double> objective, iter_seconds;
  std::vector<Params> trajectory;
};

// solver_accel.hpp:183-240 detail::run_accelerated
static Result run_accelerated(const Inputs& in, const Params& params0, const Hyper& hyper,
                              const Spec& X, const Options& opt, bool second_stage) {
  if (opt.iters < 0) throw InvalidInputError("run_accelerated: iters must be >= 0");
  Result res;
  res.params = params0;
  if (opt.compute_objective) res.objective.push_back(map_objective(in, res.params, hyper, X));
  Scratch s;
  precompute_sigma(in, X, &s);
  if (second_stage) precompute_tau(in, X, &s);
  if (second_stage)
    rho_second_stage(s, res.params.lambda, &s.rho_aa, &s.rho_ax, nullptr);
  else
    rho_first_stage(in, X, res.params.lambda, &s.rho_aa, &s.rho_ax, nullptr, opt.threads);
  Params tilde;
  for (int it = 0; it < opt.iters; ++it) {
    const auto t0 = std::chrono::steady_clock::now();
    tilde = res.params;
    s.trho_aa = s.rho_aa;
    s.trho_ax = s.rho_ax;
    compute_gamma(tilde, s.trho_aa, &s);
    if (opt.gamma_fault != 0.0)
      for (double& g : s.gamma) g += opt.gamma_fault;
    update_rh(s, tilde, hyper, opt.eps_var, &res.params.r_h);
    update_lambda(s, tilde, opt.eps_var, &res.params.lambda);
    if (second_stage)
      rho_second_stage(s, res.params.lambda, &s.rho_aa, &s.rho_ax, &s.rho_xx);
    else
      rho_first_stage(in, X, res.params.lambda, &s.rho_aa, &s.rho_ax, &s.rho_xx, opt.threads);
    update_ru(s, tilde, in.M, opt.eps_var, &res.params.r_u);
    const auto t1 = std::chrono::steady_clock::now();
    res.iter_seconds.push_back(std::chrono::duration<double>(t1 - t0).count());
    if (opt.record_trajectory) res.trajectory.push_back(res.params);
    if (opt.compute_objective) {
      res.objective.push_back(map_objective(in, res.params, hyper, X));
      const double prev = res.objective[res.objective.size() - 2];
      const double cur = res.objective.back();
      if (opt.rel_obj_tol > 0.0 && std::abs(cur - prev) <= opt.rel_obj_tol * std::abs(prev)) break;
    }
  }
  return res;
}

// Parallel second-stage iteration over bins (CPU-baseline variant). Each bin's
// arithmetic is exactly run_accelerated's (same per-bin serial t order), so the
// result is bitwise identical to the serial restatement; only independent bins
// run on different threads. Used by bench.py's reference arm with all cores.
static Result run_algorithm2_binparallel(const Inputs& in, const Params& params0,
                                         const Hyper& hyper, const Spec& X,
                                         const Options& opt) {
  if (opt.iters < 0) throw InvalidInputError("run_accelerated: iters must be >= 0");
  Result res;
  res.params = params0;
  Scratch s;
  precompute_sigma(in, X, &s);
  precompute_tau(in, X, &s);
  const Index I = X.I, J = X.J;
  const double M = static_cast<double>(in.M);
  std::vector<double> secs(opt.iters, 0.0);
  parallel_for_chunks(0, I, opt.threads, [&](Index lo, Index hi) {
    std::vector<double> rh(J), ru(J), g(J);
    std::vector<cplx> rax(J), trax(J);
    for (Index i = lo; i < hi; ++i) {
      for (Index t = 0; t < J; ++t) {
        rh[t] = params0.rh(i, t);
        ru[t] = params0.ru(i, t);
      }
      double lam = params0.lambda[i];
      double inv_lam = 1.0 / lam;
      double rho_aa = s.tau_aa[i] + std::norm(s.sigma_ab[i]) * inv_lam;
      for (Index t = 0; t < J; ++t)
        rax[t] = s.tau_ax[i + t * I] + s.sigma_ab[i] * s.sigma_bx[i + t * I] * inv_lam;
      for (int it = 0; it < opt.iters; ++it) {
        const double trho_aa = rho_aa;
        trax = rax;
        for (Index t = 0; t < J; ++t) g[t] = rh[t] / (ru[t] + rh[t] * trho_aa) + opt.gamma_fault;
        std::vector<double>& tru = ru;  // r_u is only overwritten after lambda
        const double ab2 = std::norm(s.sigma_ab[i]);
        double acc = 0.0;
        for (Index t = 0; t < J; ++t) {
          const cplx resid = s.sigma_bx[i + t * I] - g[t] * std::conj(s.sigma_ab[i]) * trax[t];
          acc += g[t] * ab2 + std::norm(resid) / tru[t];
        }
        for (Index t = 0; t < J; ++t)
          rh[t] = std::max((g[t] * (ru[t] + g[t] * std::norm(trax[t])) + hyper.beta) / (hyper.alpha + 2.0),
                           opt.eps_var);
        lam = std::max(acc / static_cast<double>(J), opt.eps_var);
        inv_lam = 1.0 / lam;
        rho_aa = s.tau_aa[i] + std::norm(s.sigma_ab[i]) * inv_lam;
        for (Index t = 0; t < J; ++t) {
          rax[t] = s.tau_ax[i + t * I] + s.sigma_ab[i] * s.sigma_bx[i + t * I] * inv_lam;
          const double rxx = s.tau_xx[i + t * I] + std::norm(s.sigma_bx[i + t * I]) * inv_lam;
          const double val = (g[t] * rho_aa * (ru[t] + g[t] * std::norm(trax[t])) + rxx -
                              2.0 * g[t] * std::real(trax[t] * std::conj(rax[t]))) / M;
          ru[t] = std::max(val, opt.eps_var);
        }
      }
      for (Index t = 0; t < J; ++t) {
        res.params.rh(i, t) = rh[t];
        res.params.ru(i, t) = ru[t];
      }
      res.params.lambda[i] = lam;
    }
  });
  (void)secs;
  return res;
}

// ---------------------------------------------------------------------------
// solver_naive.hpp
// ---------------------------------------------------------------------------

// solver_naive.hpp:46-146 closed-form Hermitian PD inverse, S in {2, 3, 4}.
static bool hermitian_pd_inverse_fixed(int S, const CMat& R, CMat* out) {
  *out = CMat(S, S);
  CMat& o = *out;
  if (S == 2) {
    const double a = std::real(R(0, 0)), c = std::real(R(1, 1));
    const cplx b = R(0, 1);
    const double det = a * c - std::norm(b);
    if (!(a > 0.0) || !(det > 0.0)) return false;
    const double inv_det = 1.0 / det;
    o(0, 0) = c * inv_det;
    o(1, 1) = a * inv_det;
    o(0, 1) = -b * inv_det;
    o(1, 0) = -std::conj(b) * inv_det;
    return true;
  }
  if (S == 3) {
    const double a = std::real(R(0, 0)), b = std::real(R(1, 1)), c = std::real(R(2, 2));
    const cplx d = R(0, 1), e = R(0, 2), f = R(1, 2);
    const double m00 = b * c - std::norm(f);
    const double m11 = a * c - std::norm(e);
    const double m22 = a * b - std::norm(d);
    const double det = std::real(a * m00 - d * (std::conj(d) * c - f * std::conj(e)) +
                                 e * (std::conj(d) * std::conj(f) - b * std::conj(e)));
    if (!(a > 0.0) || !(m22 > 0.0) || !(det > 0.0)) return false;
    const double inv_det = 1.0 / det;
    o(0, 0) = m00 * inv_det;
    o(1, 1) = m11 * inv_det;
    o(2, 2) = m22 * inv_det;
    o(0, 1) = (e * std::conj(f) - d * c) * inv_det;
    o(0, 2) = (d * f - e * b) * inv_det;
    o(1, 2) = (e * std::conj(d) - a * f) * inv_det;
    o(1, 0) = std::conj(o(0, 1));
    o(2, 0) = std::conj(o(0, 2));
    o(2, 1) = std::conj(o(1, 2));
    return true;
  }
  // S == 4: 2x2 block inversion through the Schur complement.
  const double a00 = std::real(R(0, 0)), a11 = std::real(R(1, 1));
  const cplx a01 = R(0, 1);
  const double det_a = a00 * a11 - std::norm(a01);
  if (!(a00 > 0.0) || !(det_a > 0.0)) return false;
  const double ida = 1.0 / det_a;
  const double ai00 = a11 * ida, ai11 = a00 * ida;
  const cplx ai01 = -a01 * ida, ai10 = std::conj(ai01);
  const cplx t00 = ai00 * R(0, 2) + ai01 * R(1, 2);
  const cplx t01 = ai00 * R(0, 3) + ai01 * R(1, 3);
  const cplx t10 = ai10 * R(0, 2) + ai11 * R(1, 2);
  const cplx t11 = ai10 * R(0, 3) + ai11 * R(1, 3);
  const double sc00 = std::real(R(2, 2)) - std::real(std::conj(R(0, 2)) * t00 + std::conj(R(1, 2)) * t10);
  const double sc11 = std::real(R(3, 3)) - std::real(std::conj(R(0, 3)) * t01 + std::conj(R(1, 3)) * t11);
  const cplx sc01 = R(2, 3) - std::conj(R(0, 2)) * t01 - std::conj(R(1, 2)) * t11;
  const double det_s = sc00 * sc11 - std::norm(sc01);
  if (!(sc00 > 0.0) || !(det_s > 0.0)) return false;
  const double ids = 1.0 / det_s;
  const double si00 = sc11 * ids, si11 = sc00 * ids;
  const cplx si01 = -sc01 * ids, si10 = std::conj(si01);
  const cplx u00 = t00 * si00 + t01 * si10;
  const cplx u01 = t00 * si01 + t01 * si11;
  const cplx u10 = t10 * si00 + t11 * si10;
  const cplx u11 = t10 * si01 + t11 * si11;
  o(0, 0) = ai00 + std::real(u00 * std::conj(t00) + u01 * std::conj(t01));
  o(1, 1) = ai11 + std::real(u10 * std::conj(t10) + u11 * std::conj(t11));
  o(0, 1) = ai01 + u00 * std::conj(t10) + u01 * std::conj(t11);
  o(1, 0) = std::conj(o(0, 1));
  o(0, 2) = -u00;
  o(0, 3) = -u01;
  o(1, 2) = -u10;
  o(1, 3) = -u11;
  o(2, 0) = std::conj(o(0, 2));
  o(3, 0) = std::conj(o(0, 3));
  o(2, 1) = std::conj(o(1, 2));
  o(3, 1) = std::conj(o(1, 3));
  o(2, 2) = si00;
  o(3, 3) = si11;
  o(2, 3) = si01;
  o(3, 2) = si10;
  return true;
}

static bool fixed_size(int M) { return M == 2 || M == 3 || M == 4; }

// solver_naive.hpp:153-246 naive_e_step_bin_impl (both the fixed-size and the
// dynamic LLT branch). hat_R_u_row[t] is an M x M matrix.
static void naive_e_step_bin(const Inputs& in, const Params& p, const Spec& X, Index i,
                             std::vector<double>& hat_r_h, std::vector<CMat>& hat_row) {
  const int m = X.M;
  const Index J = X.J, I = X.I;
  const CVec& a = in.a[i];
  const CVec& b = in.b[i];
  CMat Rut = in.Rp[i];
  for (int c = 0; c < m; ++c)
    for (int r = 0; r < m; ++r) Rut(r, c) += (p.lambda[i] * b[r]) * std::conj(b[c]);
  const bool fixed = fixed_size(m);
  CMat Rx(m, m), Rxi(m, m), RuRxi(m, m);
  CVec rxa(m), v(m);
  for (Index t = 0; t < J; ++t) {
    const double rh = p.rh(i, t), ru = p.ru(i, t);
    const cplx* x = X.col(i, t);
    CMat& hat = hat_row[t];
    hat = CMat(m, m);
    if (!fixed) {
      for (int c = 0; c < m; ++c)
        for (int r = 0; r < m; ++r) Rx(r, c) = (rh * a[r]) * std::conj(a[c]) + ru * Rut(r, c);
      CMat L;
      if (!llt(Rx, &L))
        throw NumericalError("e_step: singular covariance at bin " + std::to_string(i) +
                             ", frame " + std::to_string(t));
      Rxi = CMat::identity(m);
      llt_solve_inplace(L, &Rxi);
      for (int r = 0; r < m; ++r) {
        rxa[r] = 0;
        for (int k = 0; k < m; ++k) rxa[r] += Rxi(r, k) * a[k];
      }
      cplx ara = 0, xra = 0;
      for (int k = 0; k < m; ++k) {
        ara += std::conj(a[k]) * rxa[k];
        xra += std::conj(x[k]) * rxa[k];
      }
      hat_r_h[i + t * I] = rh - rh * rh * std::real(ara) + std::norm(rh * xra);
      for (int c = 0; c < m; ++c)
        for (int r = 0; r < m; ++r) {
          cplx acc = 0;
          for (int k = 0; k < m; ++k) acc += Rut(r, k) * Rxi(k, c);
          RuRxi(r, c) = acc;
        }
      for (int c = 0; c < m; ++c)
        for (int r = 0; r < m; ++r) {
          cplx acc = 0;
          for (int k = 0; k < m; ++k) acc += RuRxi(r, k) * Rut(k, c);
          hat(r, c) = -(ru * ru) * acc;
        }
      for (int c = 0; c < m; ++c)
        for (int r = 0; r < m; ++r) hat(r, c) += ru * Rut(r, c);
      for (int r = 0; r < m; ++r) {
        v[r] = 0;
        for (int k = 0; k < m; ++k) v[r] += RuRxi(r, k) * x[k];
      }
      for (int c = 0; c < m; ++c)
        for (int r = 0; r < m; ++r) hat(r, c) += ((ru * ru) * v[r]) * std::conj(v[c]);
    } else {
      for (int c = 0; c < m; ++c) {
        const cplx ac = std::conj(a[c]) * rh;
        for (int r = c; r < m; ++r) Rx(r, c) = a[r] * ac + ru * Rut(r, c);
        for (int r = 0; r < c; ++r) Rx(r, c) = std::conj(Rx(c, r));
      }
      if (!hermitian_pd_inverse_fixed(m, Rx, &Rxi))
        throw NumericalError("e_step: singular covariance at bin " + std::to_string(i) +
                             ", frame " + std::to_string(t));
      double ara = 0.0;
      cplx xra(0.0, 0.0);
      for (int r = 0; r < m; ++r) {
        cplx acc(0.0, 0.0);
        for (int c = 0; c < m; ++c) acc += Rxi(r, c) * a[c];
        rxa[r] = acc;
        ara += std::real(std::conj(a[r]) * acc);
        xra += std::conj(x[r]) * acc;
      }
      hat_r_h[i + t * I] = rh - rh * rh * ara + std::norm(rh * xra);
      for (int r = 0; r < m; ++r) {
        cplx vx(0.0, 0.0);
        for (int c = 0; c < m; ++c) {
          cplx acc(0.0, 0.0);
          for (int k = 0; k < m; ++k) acc += Rut(r, k) * Rxi(k, c);
          RuRxi(r, c) = acc;
          vx += acc * x[c];
        }
        v[r] = vx;
      }
      const double ru2 = ru * ru;
      for (int c = 0; c < m; ++c) {
        for (int r = c; r < m; ++r) {
          cplx acc(0.0, 0.0);
          for (int k = 0; k < m; ++k) acc += RuRxi(r, k) * Rut(k, c);
          hat(r, c) = ru * Rut(r, c) - ru2 * acc + ru2 * v[r] * std::conj(v[c]);
        }
        for (int r = 0; r < c; ++r) hat(r, c) = std::conj(hat(c, r));
      }
    }
  }
}

// solver_naive.hpp:267-279 e_step
static void e_step(const Inputs& in, const Params& p, const Spec& X, int threads,
                   std::vector<double>* hat_r_h, std::vector<std::vector<CMat>>* hat_R_u) {
  hat_r_h->assign(X.I * X.J, 0.0);
  hat_R_u->assign(X.I, std::vector<CMat>(X.J, CMat(X.M, X.M)));
  parallel_for_chunks(0, X.I, threads, [&](Index lo, Index hi) {
    for (Index i = lo; i < hi; ++i) naive_e_step_bin(in, p, X, i, *hat_r_h, (*hat_R_u)[i]);
  });
}

// solver_naive.hpp:282-311 m_step
static Params m_step(const std::vector<double>& hat_r_h,
                     const std::vector<std::vector<CMat>>& hat_R_u, const Inputs& in,
                     const Params& p_old, const Hyper& hyper, int threads, double eps) {
  const Index I = in.I, J = p_old.J;
  const int m = in.M;
  Params p;
  p.I = I;
  p.J = J;
  p.r_h.assign(I * J, 0.0);
  for (Index k = 0; k < I * J; ++k)
    p.r_h[k] = std::max((hat_r_h[k] + hyper.beta) / (hyper.alpha + 2.0), eps);
  p.r_u.assign(I * J, 0.0);
  p.lambda.assign(I, 0.0);
  parallel_for_chunks(0, I, threads, [&](Index lo, Index hi) {
    for (Index i = lo; i < hi; ++i) {
      const CVec& b = in.b[i];
      double lam = 0.0;
      for (Index t = 0; t < J; ++t) {
        const CMat& hat = hat_R_u[i][t];
        cplx q = 0;
        for (int r = 0; r < m; ++r) {
          cplx acc = 0;
          for (int k = 0; k < m; ++k) acc += hat(r, k) * b[k];
          q += std::conj(b[r]) * acc;
        }
        lam += std::real(q) / p_old.ru(i, t);
      }
      lam /= static_cast<double>(J);
      p.lambda[i] = std::max(lam, eps);
      CMat Ru = in.Rp[i];
      for (int c = 0; c < m; ++c)
        for (int r = 0; r < m; ++r) Ru(r, c) += (p.lambda[i] * b[r]) * std::conj(b[c]);
      CMat L;
      if (!llt(Ru, &L)) throw NumericalError("m_step: singular R^(u) at bin " + std::to_string(i));
      for (Index t = 0; t < J; ++t) {
        CMat z = hat_R_u[i][t];
        llt_solve_inplace(L, &z);
        double tr = 0;
        for (int k = 0; k < m; ++k) tr += std::real(z(k, k));
        p.ru(i, t) = std::max(tr / m, eps);
      }
    }
  });
  return p;
}

// solver_naive.hpp:319-386 naive_iteration_bin_impl (fused E/M per bin).
static void naive_iteration_bin(const Inputs& in, const Params& p_old, const Hyper& hyper,
                                const Spec& X, Index i, double eps, Params* p_new,
                                std::vector<CMat>& hat_row) {
  const Index J = X.J, I = X.I;
  const int m = X.M;
  naive_e_step_bin(in, p_old, X, i, p_new->r_h, hat_row);
  for (Index t = 0; t < J; ++t) {
    double& v = p_new->r_h[i + t * I];
    v = std::max((v + hyper.beta) / (hyper.alpha + 2.0), eps);
  }
  const CVec& b = in.b[i];
  const bool fixed = fixed_size(m);
  double lam = 0.0;
  for (Index t = 0; t < J; ++t) {
    const CMat& hat = hat_row[t];
    if (!fixed) {
      cplx q = 0;
      for (int r = 0; r < m; ++r) {
        cplx acc = 0;
        for (int k = 0; k < m; ++k) acc += hat(r, k) * b[k];
        q += std::conj(b[r]) * acc;
      }
      lam += std::real(q) / p_old.ru(i, t);
    } else {
      double q = 0.0;
      for (int c = 0; c < m; ++c) {
        q += std::real(hat(c, c)) * std::norm(b[c]);
        for (int r = c + 1; r < m; ++r) q += 2.0 * std::real(std::conj(b[r]) * hat(r, c) * b[c]);
      }
      lam += q / p_old.ru(i, t);
    }
  }
  lam /= static_cast<double>(J);
  p_new->lambda[i] = std::max(lam, eps);
  CMat Ru = in.Rp[i];
  for (int c = 0; c < m; ++c)
    for (int r = 0; r < m; ++r) Ru(r, c) += (p_new->lambda[i] * b[r]) * std::conj(b[c]);
  CMat Rui;
  if (!fixed) {
    CMat L;
    if (!llt(Ru, &L)) throw NumericalError("m_step: singular R^(u) at bin " + std::to_string(i));
    Rui = CMat::identity(m);
    llt_solve_inplace(L, &Rui);
  } else {
    if (!hermitian_pd_inverse_fixed(m, Ru, &Rui))
      throw NumericalError("m_step: singular R^(u) at bin " + std::to_string(i));
  }
  for (Index t = 0; t < J; ++t) {
    const CMat& hat = hat_row[t];
    double tr = 0.0;
    if (!fixed) {
      cplx s = 0;
      for (int c = 0; c < m; ++c)
        for (int r = 0; r < m; ++r) s += Rui(c, r) * hat(r, c);
      tr = std::real(s);
    } else {
      for (int c = 0; c < m; ++c) {
        tr += std::real(Rui(c, c)) * std::real(hat(c, c));
        for (int r = c + 1; r < m; ++r) tr += 2.0 * std::real(Rui(c, r) * hat(r, c));
      }
    }
    p_new->r_u[i + t * I] = std::max(tr / m, eps);
  }
}

// solver_naive.hpp:412-450 run_naive
static Result run_naive(const Inputs& in, const Params& params0, const Hyper& hyper,
                        const Spec& X, const Options& opt) {
  if (opt.iters < 0) throw InvalidInputError("run_naive: iters must be >= 0");
  const Index I = X.I, J = X.J;
  Result res;
  res.params = params0;
  if (opt.compute_objective) res.objective.push_back(map_objective(in, res.params, hyper, X));
  Params next;
  next.I = I;
  next.J = J;
  next.r_h.assign(I * J, 0.0);
  next.r_u.assign(I * J, 0.0);
  next.lambda.assign(I, 0.0);
  for (int it = 0; it < opt.iters; ++it) {
    const auto t0 = std::chrono::steady_clock::now();
    parallel_for_chunks(0, I, opt.threads, [&](Index lo, Index hi) {
      std::vector<CMat> hat_row(J, CMat(X.M, X.M));
      for (Index i = lo; i < hi; ++i)
        naive_iteration_bin(in, res.params, hyper, X, i, opt.eps_var, &next, hat_row);
    });
    std::swap(res.params, next);
    const auto t1 = std::chrono::steady_clock::now();
    res.iter_seconds.push_back(std::chrono::duration<double>(t1 - t0).count());
    if (opt.record_trajectory) res.trajectory.push_back(res.params);
    if (opt.compute_objective) {
      res.objective.push_back(map_objective(in, res.params, hyper, X));
      const double prev = res.objective[res.objective.size() - 2];
      const double cur = res.objective.back();
      if (opt.rel_obj_tol > 0.0 && std::abs(cur - prev) <= opt.rel_obj_tol * std::abs(prev)) break;
    }
  }
  return res;
}

// ---------------------------------------------------------------------------
// wiener.hpp
// ---------------------------------------------------------------------------

// wiener.hpp:19-43 extract_target: dry (I x J col-major), image [i][t][m].
static void extract_target(const Inputs& in, const Params& p, const Spec& X,
                           std::vector<cplx>* dry, std::vector<cplx>* image) {
  const Index I = X.I, J = X.J;
  const int m = X.M;
  Scratch s;
  precompute_sigma(in, X, &s);
  precompute_tau(in, X, &s);
  std::vector<double> rho_aa;
  std::vector<cplx> rho_ax;
  rho_second_stage(s, p.lambda, &rho_aa, &rho_ax, nullptr);
  dry->assign(I * J, 0.0);
  image->assign(I * J * m, 0.0);
  for (Index i = 0; i < I; ++i) {
    for (Index t = 0; t < J; ++t) {
      const double gamma = p.rh(i, t) / (p.ru(i, t) + p.rh(i, t) * rho_aa[i]);
      (*dry)[i + t * I] = gamma * rho_ax[i + t * I];
    }
    for (Index t = 0; t < J; ++t)
      for (int k = 0; k < m; ++k) (*image)[(i * J + t) * m + k] = in.a[i][k] * (*dry)[i + t * I];
  }
}

// ---------------------------------------------------------------------------
// verify.hpp
// ---------------------------------------------------------------------------

struct VerifyInstance {
  Inputs inputs;
  Params params;
  std::vector<cplx> X;  // [i][t][m]
};

// verify.hpp:22-56 make_verify_instance. The draw order (per bin: X col-major,
// then G col-major, then a; then per bin lambda, then (r_h, r_u) per frame)
// and cplx(gauss(engine), gauss(engine)) are kept verbatim so that, compiled
// with the same libstdc++, the instances are the reference's own.
static VerifyInstance make_verify_instance(Index bins, Index frames, int mics, uint64_t seed) {
  std::mt19937_64 engine(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  auto rand_cplx = [&] { return cplx(gauss(engine), gauss(engine)); };
  VerifyInstance inst;
  inst.X.assign(bins * frames * mics, 0.0);
  inst.inputs.I = bins;
  inst.inputs.M = mics;
  inst.inputs.n_h = 0;
  for (Index i = 0; i < bins; ++i) {
    for (Index t = 0; t < frames; ++t)
      for (int m = 0; m < mics; ++m) inst.X[(i * frames + t) * mics + m] = rand_cplx();
    CMat g(mics, mics - 1);
    for (auto& e : g.d) e = rand_cplx();
    CMat rp(mics, mics);
    for (int c = 0; c < mics; ++c)
      for (int r = 0; r < mics; ++r) {
        cplx s = 0;
        for (int k = 0; k < mics - 1; ++k) s += g(r, k) * std::conj(g(c, k));
        rp(r, c) = s;
      }
    CMat sym(mics, mics);
    for (int c = 0; c < mics; ++c)
      for (int r = 0; r < mics; ++r) sym(r, c) = (rp(r, c) + std::conj(rp(c, r))) / 2.0;
    inst.inputs.Rp.push_back(sym);
    inst.inputs.Rpp.push_back(pseudo_inverse_psd(sym));
    inst.inputs.b.push_back(null_eigenvector(sym));
    CVec a(mics);
    for (auto& e : a) e = rand_cplx();
    inst.inputs.a.push_back(a);
  }
  inst.params.I = bins;
  inst.params.J = frames;
  inst.params.r_h.assign(bins * frames, 0.0);
  inst.params.r_u.assign(bins * frames, 0.0);
  inst.params.lambda.assign(bins, 0.0);
  for (Index i = 0; i < bins; ++i) {
    inst.params.lambda[i] = 0.1 + std::abs(gauss(engine));
    for (Index t = 0; t < frames; ++t) {
      inst.params.rh(i, t) = 0.1 + std::abs(gauss(engine));
      inst.params.ru(i, t) = 0.1 + std::abs(gauss(engine));
    }
  }
  return inst;
}

// verify.hpp:60-68
static double rel_dist(const double* x, const double* y, Index n) {
  double worst = 0;
  for (Index k = 0; k < n; ++k) {
    const double den = std::max({std::abs(x[k]), std::abs(y[k]), kEpsVar});
    worst = std::max(worst, std::abs(x[k] - y[k]) / den);
  }
  return worst;
}

// ===========================================================================
// ilrma.hpp: sphering, Gaussian ILRMA (IP + NMF), objective
// ===========================================================================

constexpr double kNmfVarFloor = 1e-12;  // ilrma.hpp:40

// Eigen::FullPivLU semantics (complete pivoting; pivot = first maximum |a_ij|
// in column-major order of the remaining corner; rank counts pivots above
// M * eps * |max pivot|), for the IP solve and the final inverse.
struct FullPivLU {
  int n = 0;
  CMat lu;
  std::vector<int> rowp, colp;  // row / column transpositions
  int nonzero = 0;
  double maxpivot = 0.0;
  explicit FullPivLU(const CMat& A) : n(A.rows), lu(A), rowp(A.rows), colp(A.rows) {
    nonzero = n;
    for (int k = 0; k < n; ++k) {
      int br = k, bc = k;
      double big = -1.0;
      for (int c = k; c < n; ++c)
        for (int r = k; r < n; ++r) {
          const double v = std::abs(lu(r, c));
          if (v > big) {
            big = v;
            br = r;
            bc = c;
          }
        }
      if (big == 0.0) {
        nonzero = k;
        for (int i = k; i < n; ++i) rowp[i] = colp[i] = i;
        break;
      }
      if (big > maxpivot) maxpivot = big;
      rowp[k] = br;
      colp[k] = bc;
      if (br != k)
        for (int c = 0; c < n; ++c) std::swap(lu(k, c), lu(br, c));
      if (bc != k)
        for (int r = 0; r < n; ++r) std::swap(lu(r, k), lu(r, bc));
      for (int r = k + 1; r < n; ++r) lu(r, k) /= lu(k, k);
      for (int c = k + 1; c < n; ++c)
        for (int r = k + 1; r < n; ++r) lu(r, c) -= lu(r, k) * lu(k, c);
    }
  }
  int rank() const {
    const double thr = n * std::numeric_limits<double>::epsilon() * maxpivot;
    int rk = 0;
    for (int i = 0; i < nonzero; ++i) rk += std::abs(lu(i, i)) > thr;
    return rk;
  }
  bool invertible() const { return rank() == n; }
  CVec solve(const CVec& b) const {  // A x = b for invertible A
    CVec y = b;
    for (int k = 0; k < n; ++k) std::swap(y[k], y[rowp[k]]);
    for (int r = 0; r < n; ++r)
      for (int c = 0; c < r; ++c) y[r] -= lu(r, c) * y[c];
    for (int r = n - 1; r >= 0; --r) {
      for (int c = r + 1; c < n; ++c) y[r] -= lu(r, c) * y[c];
      y[r] /= lu(r, r);
    }
    for (int k = n - 1; k >= 0; --k) std::swap(y[k], y[colp[k]]);
    return y;
  }
  CMat inverse() const {
    CMat out(n, n);
    for (int c = 0; c < n; ++c) {
      CVec e(n, cplx(0, 0));
      e[c] = 1.0;
      const CVec x = solve(e);
      for (int r = 0; r < n; ++r) out(r, c) = x[r];
    }
    return out;
  }
};

static CMat matmul(const CMat& A, const CMat& B) {
  CMat C(A.rows, B.cols);
  for (int c = 0; c < B.cols; ++c)
    for (int k = 0; k < A.cols; ++k)
      for (int r = 0; r < A.rows; ++r) C(r, c) += A(r, k) * B(k, c);
  return C;
}

// ilrma.hpp:53-73 sphere: per bin cov = X X^H / J + (1e-10 tr/M) I,
// Q = sum_k v_k v_k^H / sqrt(max(l_k, 1e-300)) of eig((cov + cov^H)/2), Xw = Q X.
static void sphere(const Spec& X, std::vector<CMat>* Q, std::vector<cplx>* Xw) {
  const int m = X.M;
  const Index j = X.J;
  if (j <= m) throw InvalidInputError("sphere: need more frames than channels");
  Q->assign(X.I, CMat());
  Xw->assign(static_cast<size_t>(X.I * j * m), cplx(0, 0));
  for (Index i = 0; i < X.I; ++i) {
    CMat cov(m, m);
    for (Index t = 0; t < j; ++t) {
      const cplx* x = X.col(i, t);
      for (int c = 0; c < m; ++c)
        for (int r = 0; r < m; ++r) cov(r, c) += x[r] * std::conj(x[c]);
    }
    double tr = 0.0;
    for (int r = 0; r < m; ++r) tr += std::real(cov(r, r) / static_cast<double>(j));
    for (auto& v : cov.d) v /= static_cast<double>(j);
    for (int r = 0; r < m; ++r) cov(r, r) += 1e-10 * tr / m;
    CMat h(m, m);
    for (int c = 0; c < m; ++c)
      for (int r = 0; r < m; ++r) h(r, c) = (cov(r, c) + std::conj(cov(c, r))) / 2.0;
    const EigResult eig = hermitian_eig(h);
    CMat q(m, m);
    for (int k = 0; k < m; ++k) {
      const double l = std::max(eig.values[k], 1e-300);
      const double s = 1.0 / std::sqrt(l);
      for (int c = 0; c < m; ++c)
        for (int r = 0; r < m; ++r) q(r, c) += s * eig.vectors(r, k) * std::conj(eig.vectors(c, k));
    }
    (*Q)[i] = q;
    for (Index t = 0; t < j; ++t) {
      const cplx* x = X.col(i, t);
      cplx* y = Xw->data() + (i * j + t) * m;
      for (int r = 0; r < m; ++r)
        for (int c = 0; c < m; ++c) y[r] += q(r, c) * x[c];
    }
  }
}

struct Nmf {  // ilrma.hpp:26-29: per source T (I x K), V (K x J), column-major
  std::vector<std::vector<double>> T, V;
};

// ilrma.hpp:100-123
static void nmf_update(const std::vector<std::vector<double>>& P, Index I, Index J, int K, Nmf* nmf) {
  const size_t ns = P.size();
  std::vector<double> R(I * J), PR2(I * J), Rinv(I * J);
  auto model = [&](const std::vector<double>& T, const std::vector<double>& V) {
    for (Index t = 0; t < J; ++t)
      for (Index i = 0; i < I; ++i) {
        double s = 0.0;
        for (int k = 0; k < K; ++k) s += T[i + k * I] * V[k + t * K];
        const double r = std::max(s, kNmfVarFloor);
        R[i + t * I] = r;
      }
  };
  for (size_t n = 0; n < ns; ++n) {
    std::vector<double>& T = nmf->T[n];
    std::vector<double>& V = nmf->V[n];
    const std::vector<double>& Pn = P[n];
    model(T, V);
    for (Index e = 0; e < I * J; ++e) {
      PR2[e] = Pn[e] / (R[e] * R[e]);
      Rinv[e] = 1.0 / R[e];
    }
    std::vector<double> Tn(T.size());
    for (int k = 0; k < K; ++k)
      for (Index i = 0; i < I; ++i) {
        double num = 0.0, den = 0.0;
        for (Index t = 0; t < J; ++t) {
          num += PR2[i + t * I] * V[k + t * K];
          den += Rinv[i + t * I] * V[k + t * K];
        }
        Tn[i + k * I] = std::max(T[i + k * I] * std::sqrt(num / std::max(den, 1e-300)), 1e-300);
      }
    T = Tn;
    model(T, V);
    for (Index e = 0; e < I * J; ++e) {
      PR2[e] = Pn[e] / (R[e] * R[e]);
      Rinv[e] = 1.0 / R[e];
    }
    std::vector<double> Vn(V.size());
    for (Index t = 0; t < J; ++t)
      for (int k = 0; k < K; ++k) {
        double num = 0.0, den = 0.0;
        for (Index i = 0; i < I; ++i) {
          num += T[i + k * I] * PR2[i + t * I];
          den += T[i + k * I] * Rinv[i + t * I];
        }
        Vn[k + t * K] = std::max(V[k + t * K] * std::sqrt(num / std::max(den, 1e-300)), 1e-300);
      }
    V = Vn;
  }
}

// ilrma.hpp:125-135: P[n](i, t) = |(W_i x_it)_n|^2
static void demixed_powers(const std::vector<CMat>& W, const Spec& X, std::vector<std::vector<double>>* P) {
  const int m = X.M;
  for (Index i = 0; i < X.I; ++i)
    for (Index t = 0; t < X.J; ++t) {
      const cplx* x = X.col(i, t);
      for (int n = 0; n < m; ++n) {
        cplx y(0, 0);
        for (int c = 0; c < m; ++c) y += W[i](n, c) * x[c];
        (*P)[n][i + t * X.I] = std::norm(y);
      }
    }
}

// ilrma.hpp:145-240 run_ilrma
static void run_ilrma(const Spec& X, int K, int iters, uint64_t seed, std::vector<CMat>* Wout,
                      std::vector<CMat>* Aout, Nmf* nmf) {
  const Index I = X.I, J = X.J;
  const int m = X.M;
  if (K < 1) throw InvalidInputError("run_ilrma: K must be >= 1");
  if (iters < 0) throw InvalidInputError("run_ilrma: iters must be >= 0");
  std::vector<CMat> W(I, CMat::identity(m));
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unif(0.1, 1.0);
  nmf->T.assign(m, std::vector<double>());
  nmf->V.assign(m, std::vector<double>());
  for (int n = 0; n < m; ++n) {
    nmf->T[n].assign(I * K, 0.0);
    nmf->V[n].assign(static_cast<size_t>(K) * J, 0.0);
    for (Index i = 0; i < I; ++i)
      for (int k = 0; k < K; ++k) nmf->T[n][i + k * I] = unif(rng);
    for (int k = 0; k < K; ++k)
      for (Index t = 0; t < J; ++t) nmf->V[n][k + t * K] = unif(rng);
  }
  std::vector<std::vector<double>> P(m, std::vector<double>(I * J, 0.0));
  demixed_powers(W, X, &P);
  for (int pass = 0; pass < 30; ++pass) nmf_update(P, I, J, K, nmf);
  for (int it = 0; it < iters; ++it) {
    nmf_update(P, I, J, K, nmf);
    std::vector<std::vector<double>> Rinv(m, std::vector<double>(I * J));
    for (int n = 0; n < m; ++n)
      for (Index t = 0; t < J; ++t)
        for (Index i = 0; i < I; ++i) {
          double s = 0.0;
          for (int k = 0; k < K; ++k) s += nmf->T[n][i + k * I] * nmf->V[n][k + t * K];
          Rinv[n][i + t * I] = 1.0 / std::max(s, kNmfVarFloor);
        }
    for (Index i = 0; i < I; ++i) {
      CMat& Wi = W[i];
      for (int n = 0; n < m; ++n) {
        CMat U(m, m);
        for (Index t = 0; t < J; ++t) {
          const cplx* x = X.col(i, t);
          const double w = Rinv[n][i + t * I];
          for (int c = 0; c < m; ++c)
            for (int r = 0; r < m; ++r) U(r, c) += w * x[r] * std::conj(x[c]);
        }
        for (auto& v : U.d) v /= static_cast<double>(J);
        CMat WU = matmul(Wi, U);
        FullPivLU lu(WU);
        if (!lu.invertible()) {
          double nrm = 0.0;
          for (const auto& v : WU.d) nrm += std::norm(v);
          const double load = 1e-8 * std::max(std::sqrt(nrm), 1e-30);
          for (int r = 0; r < m; ++r) WU(r, r) += load;
          lu = FullPivLU(WU);
          if (!lu.invertible())
            throw NumericalError("run_ilrma: singular spatial update at frequency bin " + std::to_string(i));
        }
        CVec e(m, cplx(0, 0));
        e[n] = 1.0;
        CVec w = lu.solve(e);
        cplx uw_dot(0, 0);
        for (int r = 0; r < m; ++r) {
          cplx uw(0, 0);
          for (int c = 0; c < m; ++c) uw += U(r, c) * w[c];
          uw_dot += std::conj(w[r]) * uw;
        }
        const double s = std::sqrt(std::max(std::real(uw_dot), 1e-300));
        for (int c = 0; c < m; ++c) Wi(n, c) = std::conj(w[c] / s);
      }
    }
    demixed_powers(W, X, &P);
    for (int n = 0; n < m; ++n) {
      double sum = 0.0;
      for (double v : P[n]) sum += v;
      const double mu = std::sqrt(sum / static_cast<double>(I * J));
      if (mu > 0.0 && std::isfinite(mu)) {
        for (Index i = 0; i < I; ++i)
          for (int c = 0; c < m; ++c) W[i](n, c) /= mu;
        for (double& v : P[n]) v /= mu * mu;
        for (double& v : nmf->T[n]) v /= mu * mu;
      }
    }
  }
  Aout->assign(I, CMat());
  for (Index i = 0; i < I; ++i) {
    FullPivLU lu(W[i]);
    if (!lu.invertible())
      throw NumericalError("run_ilrma: singular demixing matrix at frequency bin " + std::to_string(i));
    (*Aout)[i] = lu.inverse();
  }
  *Wout = W;
}

// ilrma.hpp:86-98 ilrma_objective (|det W| by complete-pivoting LU)
static double ilrma_objective(const std::vector<CMat>& W, const Nmf& nmf, int K, const Spec& X) {
  const Index I = X.I, J = X.J;
  const int m = X.M;
  double obj = 0.0;
  for (Index i = 0; i < I; ++i) {
    for (int n = 0; n < m; ++n)
      for (Index t = 0; t < J; ++t) {
        double s = 0.0;
        for (int k = 0; k < K; ++k) s += nmf.T[n][i + k * I] * nmf.V[n][k + t * K];
        const double r = std::max(s, kNmfVarFloor);
        const cplx* x = X.col(i, t);
        cplx y(0, 0);
        for (int c = 0; c < m; ++c) y += W[i](n, c) * x[c];
        obj += std::norm(y) / r + std::log(r);
      }
    FullPivLU lu(W[i]);
    cplx det(1.0, 0.0);
    for (int k = 0; k < m; ++k) det *= lu.lu(k, k);
    int swaps = 0;
    for (int k = 0; k < m; ++k) swaps += (lu.rowp[k] != k) + (lu.colp[k] != k);
    if (swaps % 2) det = -det;
    obj -= 2.0 * J * std::log(std::abs(det) + 1e-300);
  }
  return obj;
}

}  // namespace oracle

// ===========================================================================
// C ABI
// ===========================================================================

using namespace oracle;

static thread_local std::string g_last_error;

template <class F>
static int guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return 0;
  } catch (const InvalidInputError& e) {
    g_last_error = e.what();
    return 2;
  } catch (const NumericalError& e) {
    g_last_error = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return 5;
  }
}

static std::vector<CMat> load_mats(const double* p, Index I, int M) {
  std::vector<CMat> v(I);
  for (Index i = 0; i < I; ++i) v[i] = load_mat(p + 2 * i * M * M, M);
  return v;
}
static Spec make_spec(Index I, Index J, int M, const double* X) {
  Spec s;
  s.I = I;
  s.J = J;
  s.M = M;
  s.x = C(X);
  return s;
}
static void store_params(const Params& p, double* r_h, double* r_u, double* lam) {
  if (r_h) std::memcpy(r_h, p.r_h.data(), sizeof(double) * p.r_h.size());
  if (r_u) std::memcpy(r_u, p.r_u.data(), sizeof(double) * p.r_u.size());
  if (lam) std::memcpy(lam, p.lambda.data(), sizeof(double) * p.lambda.size());
}

extern "C" {

const char* oracle_last_error(void) { return g_last_error.c_str(); }

int oracle_hermitian_eig(int M, const double* H, double* values, double* vectors) {
  return guarded([&] {
    const EigResult e = hermitian_eig(load_mat(H, M));
    std::memcpy(values, e.values.data(), sizeof(double) * M);
    store_mat(e.vectors, vectors);
  });
}
int oracle_pseudo_inverse_psd(int M, const double* H, double rank_tol, double* out) {
  return guarded([&] { store_mat(pseudo_inverse_psd(load_mat(H, M), rank_tol), out); });
}
int oracle_null_eigenvector(int M, const double* H, double rank_tol, double* out) {
  return guarded([&] {
    const CVec v = null_eigenvector(load_mat(H, M), rank_tol);
    std::memcpy(out, v.data(), sizeof(cplx) * M);
  });
}
int oracle_normalize_phase(int M, const double* v, double* out) {
  return guarded([&] {
    const CVec r = normalize_phase(load_vec(v, M));
    std::memcpy(out, r.data(), sizeof(cplx) * M);
  });
}
int oracle_sherman_morrison_inverse(int M, const double* Rinv, const double* a, double c,
                                    double d, double* out) {
  return guarded(
      [&] { store_mat(sherman_morrison_inverse(load_mat(Rinv, M), load_vec(a, M), c, d), out); });
}
int oracle_rank_one_restored_inverse(int M, const double* Rpp, const double* b, double lambda,
                                     double* out) {
  return guarded(
      [&] { store_mat(rank_one_restored_inverse(load_mat(Rpp, M), load_vec(b, M), lambda), out); });
}

int oracle_build_noise_scm(int64_t I, int64_t J, int M, const double* X, const double* W,
                           const double* A, int n_h, double rank_tol, double* a, double* Rp,
                           double* Rpp, double* b) {
  return guarded([&] {
    Inputs in;
    build_noise_scm(load_mats(W, I, M), load_mats(A, I, M), make_spec(I, J, M, X), n_h, rank_tol,
                    &in);
    for (Index i = 0; i < I; ++i) {
      std::memcpy(a + 2 * i * M, in.a[i].data(), sizeof(cplx) * M);
      std::memcpy(b + 2 * i * M, in.b[i].data(), sizeof(cplx) * M);
      store_mat(in.Rp[i], Rp + 2 * i * M * M);
      store_mat(in.Rpp[i], Rpp + 2 * i * M * M);
    }
  });
}

int oracle_init_params(int64_t I, int64_t J, int M, int K, const double* X, const double* W,
                       const double* A, int n_h, const double* Rp, const double* Rpp,
                       const double* T, const double* V, double* r_h, double* r_u,
                       double* lambda) {
  return guarded([&] {
    Inputs in = make_inputs(I, M, nullptr, Rp, Rpp, nullptr);
    in.n_h = n_h;
    Params p;
    init_params(in, T, V, K, load_mats(W, I, M), load_mats(A, I, M), make_spec(I, J, M, X), &p);
    store_params(p, r_h, r_u, lambda);
  });
}

int oracle_map_objective(int64_t I, int64_t J, int M, const double* a, const double* Rp,
                         const double* b, const double* r_h, const double* r_u,
                         const double* lambda, double alpha, double beta, const double* X,
                         double* out) {
  return guarded([&] {
    const Inputs in = make_inputs(I, M, a, Rp, nullptr, b);
    const Params p = make_params(I, J, r_h, r_u, lambda);
    *out = map_objective(in, p, Hyper{alpha, beta}, make_spec(I, J, M, X));
  });
}

int oracle_precompute(int64_t I, int64_t J, int M, const double* a, const double* Rpp,
                      const double* b, const double* X, double* sigma_ab, double* sigma_bx,
                      double* tau_aa, double* tau_ax, double* tau_xx) {
  return guarded([&] {
    const Inputs in = make_inputs(I, M, a, nullptr, Rpp, b);
    const Spec x = make_spec(I, J, M, X);
    Scratch s;
    precompute_sigma(in, x, &s);
    precompute_tau(in, x, &s);
    std::memcpy(sigma_ab, s.sigma_ab.data(), sizeof(cplx) * I);
    std::memcpy(sigma_bx, s.sigma_bx.data(), sizeof(cplx) * I * J);
    std::memcpy(tau_aa, s.tau_aa.data(), sizeof(double) * I);
    std::memcpy(tau_ax, s.tau_ax.data(), sizeof(cplx) * I * J);
    std::memcpy(tau_xx, s.tau_xx.data(), sizeof(double) * I * J);
  });
}

int oracle_compute_gamma(int64_t I, int64_t J, const double* r_h, const double* r_u,
                         const double* trho_aa, double* gamma) {
  return guarded([&] {
    Params t;
    t.I = I;
    t.J = J;
    t.r_h.assign(r_h, r_h + I * J);
    t.r_u.assign(r_u, r_u + I * J);
    Scratch s;
    compute_gamma(t, std::vector<double>(trho_aa, trho_aa + I), &s);
    std::memcpy(gamma, s.gamma.data(), sizeof(double) * I * J);
  });
}

int oracle_rho_first_stage(int64_t I, int64_t J, int M, const double* Rp, const double* a,
                           const double* b, const double* X, const double* lambda,
                           double* rho_aa, double* rho_ax, double* rho_xx) {
  return guarded([&] {
    const Inputs in = make_inputs(I, M, a, Rp, nullptr, b);
    std::vector<double> raa, rxx;
    std::vector<cplx> rax;
    rho_first_stage(in, make_spec(I, J, M, X), std::vector<double>(lambda, lambda + I), &raa,
                    &rax, rho_xx ? &rxx : nullptr, 1);
    std::memcpy(rho_aa, raa.data(), sizeof(double) * I);
    std::memcpy(rho_ax, rax.data(), sizeof(cplx) * I * J);
    if (rho_xx) std::memcpy(rho_xx, rxx.data(), sizeof(double) * I * J);
  });
}

static Scratch make_scratch(int64_t I, int64_t J, const double* sigma_ab, const double* sigma_bx,
                            const double* tau_aa, const double* tau_ax, const double* tau_xx) {
  Scratch s;
  s.I = I;
  s.J = J;
  if (sigma_ab) s.sigma_ab.assign(C(sigma_ab), C(sigma_ab) + I);
  if (sigma_bx) s.sigma_bx.assign(C(sigma_bx), C(sigma_bx) + I * J);
  if (tau_aa) s.tau_aa.assign(tau_aa, tau_aa + I);
  if (tau_ax) s.tau_ax.assign(C(tau_ax), C(tau_ax) + I * J);
  if (tau_xx) s.tau_xx.assign(tau_xx, tau_xx + I * J);
  return s;
}

int oracle_rho_second_stage(int64_t I, int64_t J, const double* sigma_ab, const double* sigma_bx,
                            const double* tau_aa, const double* tau_ax, const double* tau_xx,
                            const double* lambda, double* rho_aa, double* rho_ax,
                            double* rho_xx) {
  return guarded([&] {
    const Scratch s = make_scratch(I, J, sigma_ab, sigma_bx, tau_aa, tau_ax, tau_xx);
    std::vector<double> raa, rxx;
    std::vector<cplx> rax;
    rho_second_stage(s, std::vector<double>(lambda, lambda + I), &raa, &rax,
                     rho_xx ? &rxx : nullptr);
    std::memcpy(rho_aa, raa.data(), sizeof(double) * I);
    std::memcpy(rho_ax, rax.data(), sizeof(cplx) * I * J);
    if (rho_xx) std::memcpy(rho_xx, rxx.data(), sizeof(double) * I * J);
  });
}

int oracle_update_rh(int64_t I, int64_t J, const double* gamma, const double* r_u,
                     const double* trho_ax, double alpha, double beta, double eps,
                     double* r_h_out) {
  return guarded([&] {
    Scratch s;
    s.gamma.assign(gamma, gamma + I * J);
    s.trho_ax.assign(C(trho_ax), C(trho_ax) + I * J);
    Params t;
    t.I = I;
    t.J = J;
    t.r_u.assign(r_u, r_u + I * J);
    std::vector<double> out;
    update_rh(s, t, Hyper{alpha, beta}, eps, &out);
    std::memcpy(r_h_out, out.data(), sizeof(double) * I * J);
  });
}

int oracle_update_lambda(int64_t I, int64_t J, const double* gamma, const double* r_u,
                         const double* sigma_ab, const double* sigma_bx, const double* trho_ax,
                         double eps, double* lambda_out) {
  return guarded([&] {
    Scratch s = make_scratch(I, J, sigma_ab, sigma_bx, nullptr, nullptr, nullptr);
    s.gamma.assign(gamma, gamma + I * J);
    s.trho_ax.assign(C(trho_ax), C(trho_ax) + I * J);
    Params t;
    t.I = I;
    t.J = J;
    t.r_u.assign(r_u, r_u + I * J);
    std::vector<double> out;
    update_lambda(s, t, eps, &out);
    std::memcpy(lambda_out, out.data(), sizeof(double) * I);
  });
}

int oracle_update_ru(int64_t I, int64_t J, int M, const double* gamma, const double* r_u,
                     const double* rho_aa, const double* rho_ax, const double* trho_ax,
                     const double* rho_xx, double eps, double* r_u_out) {
  return guarded([&] {
    Scratch s;
    s.I = I;
    s.J = J;
    s.gamma.assign(gamma, gamma + I * J);
    s.rho_aa.assign(rho_aa, rho_aa + I);
    s.rho_ax.assign(C(rho_ax), C(rho_ax) + I * J);
    s.trho_ax.assign(C(trho_ax), C(trho_ax) + I * J);
    s.rho_xx.assign(rho_xx, rho_xx + I * J);
    Params t;
    t.I = I;
    t.J = J;
    t.r_u.assign(r_u, r_u + I * J);
    std::vector<double> out;
    update_ru(s, t, M, eps, &out);
    std::memcpy(r_u_out, out.data(), sizeof(double) * I * J);
  });
}

int oracle_hermitian_pd_inverse(int M, const double* R, double* out) {
  return guarded([&] {
    const CMat r = load_mat(R, M);
    CMat o;
    bool ok;
    if (fixed_size(M)) {
      ok = hermitian_pd_inverse_fixed(M, r, &o);
    } else {
      CMat L;
      ok = llt(r, &L);
      if (ok) {
        o = CMat::identity(M);
        llt_solve_inplace(L, &o);
      }
    }
    if (!ok) throw NumericalError("hermitian_pd_inverse: matrix is not positive definite");
    store_mat(o, out);
  });
}

int oracle_e_step(int64_t I, int64_t J, int M, const double* a, const double* Rp,
                  const double* b, const double* r_h, const double* r_u, const double* lambda,
                  const double* X, double* hat_r_h, double* hat_R_u) {
  return guarded([&] {
    const Inputs in = make_inputs(I, M, a, Rp, nullptr, b);
    const Params p = make_params(I, J, r_h, r_u, lambda);
    std::vector<double> hr;
    std::vector<std::vector<CMat>> hu;
    e_step(in, p, make_spec(I, J, M, X), 1, &hr, &hu);
    std::memcpy(hat_r_h, hr.data(), sizeof(double) * I * J);
    for (Index i = 0; i < I; ++i)
      for (Index t = 0; t < J; ++t) store_mat(hu[i][t], hat_R_u + 2 * (i * J + t) * M * M);
  });
}

int oracle_m_step(int64_t I, int64_t J, int M, const double* hat_r_h, const double* hat_R_u,
                  const double* Rp, const double* b, const double* r_u_old, double alpha,
                  double beta, double eps, double* r_h, double* r_u, double* lambda) {
  return guarded([&] {
    const Inputs in = make_inputs(I, M, nullptr, Rp, nullptr, b);
    Params old;
    old.I = I;
    old.J = J;
    old.r_u.assign(r_u_old, r_u_old + I * J);
    std::vector<std::vector<CMat>> hu(I, std::vector<CMat>(J));
    for (Index i = 0; i < I; ++i)
      for (Index t = 0; t < J; ++t) hu[i][t] = load_mat(hat_R_u + 2 * (i * J + t) * M * M, M);
    const Params p = m_step(std::vector<double>(hat_r_h, hat_r_h + I * J), hu, in, old,
                            Hyper{alpha, beta}, 1, eps);
    store_params(p, r_h, r_u, lambda);
  });
}

int oracle_run(int backend, int64_t I, int64_t J, int M, const double* a, const double* Rp,
               const double* Rpp, const double* b, const double* r_h0, const double* r_u0,
               const double* lambda0, double alpha, double beta, const double* X,
               const oracle_solver_opts* o, double* r_h, double* r_u, double* lambda,
               double* objective, int* n_obj, double* iter_seconds, int* n_iter,
               double* traj_r_h, double* traj_r_u, double* traj_lambda) {
  return guarded([&] {
    Inputs in = make_inputs(I, M, a, Rp, Rpp, b);
    const Params p0 = make_params(I, J, r_h0, r_u0, lambda0);
    Options opt;
    opt.iters = o->iters;
    opt.compute_objective = o->compute_objective != 0;
    opt.record_trajectory = o->record_trajectory != 0;
    opt.rel_obj_tol = o->rel_obj_tol;
    opt.threads = o->threads;
    opt.eps_var = o->eps_var;
    opt.gamma_fault = o->gamma_fault;
    const Hyper h{alpha, beta};
    const Spec x = make_spec(I, J, M, X);
    Result res;
    if (backend == 0)
      res = run_naive(in, p0, h, x, opt);
    else if (backend == 1)
      res = run_accelerated(in, p0, h, x, opt, false);
    else if (backend == 2)
      res = run_accelerated(in, p0, h, x, opt, true);
    else if (backend == 3)  // bin-parallel second stage (CPU baseline, all cores)
      res = run_algorithm2_binparallel(in, p0, h, x, opt);
    else
      throw InvalidInputError("oracle_run: unknown backend");
    store_params(res.params, r_h, r_u, lambda);
    if (n_obj) *n_obj = static_cast<int>(res.objective.size());
    if (objective)
      std::memcpy(objective, res.objective.data(), sizeof(double) * res.objective.size());
    if (n_iter) *n_iter = static_cast<int>(res.iter_seconds.size());
    if (iter_seconds)
      std::memcpy(iter_seconds, res.iter_seconds.data(), sizeof(double) * res.iter_seconds.size());
    for (size_t k = 0; k < res.trajectory.size(); ++k) {
      if (traj_r_h) std::memcpy(traj_r_h + k * I * J, res.trajectory[k].r_h.data(), sizeof(double) * I * J);
      if (traj_r_u) std::memcpy(traj_r_u + k * I * J, res.trajectory[k].r_u.data(), sizeof(double) * I * J);
      if (traj_lambda) std::memcpy(traj_lambda + k * I, res.trajectory[k].lambda.data(), sizeof(double) * I);
    }
  });
}

int oracle_extract_target(int64_t I, int64_t J, int M, const double* a, const double* Rpp,
                          const double* b, const double* r_h, const double* r_u,
                          const double* lambda, const double* X, double* image, double* dry) {
  return guarded([&] {
    const Inputs in = make_inputs(I, M, a, nullptr, Rpp, b);
    const Params p = make_params(I, J, r_h, r_u, lambda);
    std::vector<cplx> d, img;
    extract_target(in, p, make_spec(I, J, M, X), &d, &img);
    if (dry) std::memcpy(dry, d.data(), sizeof(cplx) * I * J);
    if (image) std::memcpy(image, img.data(), sizeof(cplx) * I * J * M);
  });
}

int oracle_extract_noise(int64_t I, int64_t J, int M, const double* a, const double* Rpp,
                         const double* b, const double* r_h, const double* r_u,
                         const double* lambda, const double* X, double* noise) {
  return guarded([&] {
    const Inputs in = make_inputs(I, M, a, nullptr, Rpp, b);
    const Params p = make_params(I, J, r_h, r_u, lambda);
    std::vector<cplx> d, img;
    extract_target(in, p, make_spec(I, J, M, X), &d, &img);
    const cplx* x = C(X);
    cplx* out = C(noise);
    for (Index k = 0; k < I * J * M; ++k) out[k] = x[k] - img[k];  // wiener.hpp:46-53
  });
}

int oracle_make_verify_instance(int64_t I, int64_t J, int M, uint64_t seed, double* X, double* a,
                                double* Rp, double* Rpp, double* b, double* r_h, double* r_u,
                                double* lambda) {
  return guarded([&] {
    const VerifyInstance inst = make_verify_instance(I, J, M, seed);
    std::memcpy(X, inst.X.data(), sizeof(cplx) * I * J * M);
    for (Index i = 0; i < I; ++i) {
      std::memcpy(a + 2 * i * M, inst.inputs.a[i].data(), sizeof(cplx) * M);
      std::memcpy(b + 2 * i * M, inst.inputs.b[i].data(), sizeof(cplx) * M);
      store_mat(inst.inputs.Rp[i], Rp + 2 * i * M * M);
      store_mat(inst.inputs.Rpp[i], Rpp + 2 * i * M * M);
    }
    store_params(inst.params, r_h, r_u, lambda);
  });
}

double oracle_trajectory_distance(int64_t I, int64_t J, const double* r_h_a, const double* r_u_a,
                                  const double* lam_a, const double* r_h_b, const double* r_u_b,
                                  const double* lam_b) {
  return std::max({rel_dist(r_h_a, r_h_b, I * J), rel_dist(r_u_a, r_u_b, I * J),
                   rel_dist(lam_a, lam_b, I)});
}

// ilrma.hpp:53-73 (Q: [i][M*M] col-major, Xw: [i][t][m])
int oracle_sphere(int64_t I, int64_t J, int M, const double* X, double* Q, double* Xw) {
  return guarded([&] {
    std::vector<CMat> q;
    std::vector<cplx> xw;
    sphere(make_spec(I, J, M, X), &q, &xw);
    for (Index i = 0; i < I; ++i) store_mat(q[i], Q + 2 * i * M * M);
    std::memcpy(Xw, xw.data(), sizeof(cplx) * xw.size());
  });
}

// ilrma.hpp:145-240 (W, A: [i][M*M]; T: [n][I x K col-major]; V: [n][K x J col-major])
int oracle_run_ilrma(int64_t I, int64_t J, int M, int K, int iters, uint64_t seed, const double* X, double* W,
                     double* A, double* T, double* V) {
  return guarded([&] {
    std::vector<CMat> w, a;
    Nmf nmf;
    run_ilrma(make_spec(I, J, M, X), K, iters, seed, &w, &a, &nmf);
    for (Index i = 0; i < I; ++i) {
      store_mat(w[i], W + 2 * i * M * M);
      store_mat(a[i], A + 2 * i * M * M);
    }
    for (int n = 0; n < M; ++n) {
      std::memcpy(T + static_cast<size_t>(n) * I * K, nmf.T[n].data(), sizeof(double) * I * K);
      std::memcpy(V + static_cast<size_t>(n) * K * J, nmf.V[n].data(), sizeof(double) * K * J);
    }
  });
}

// ilrma.hpp:86-98
int oracle_ilrma_objective(int64_t I, int64_t J, int M, int K, const double* X, const double* W, const double* T,
                           const double* V, double* out) {
  return guarded([&] {
    Nmf nmf;
    nmf.T.resize(M);
    nmf.V.resize(M);
    for (int n = 0; n < M; ++n) {
      nmf.T[n].assign(T + static_cast<size_t>(n) * I * K, T + static_cast<size_t>(n + 1) * I * K);
      nmf.V[n].assign(V + static_cast<size_t>(n) * K * J, V + static_cast<size_t>(n + 1) * K * J);
    }
    *out = ilrma_objective(load_mats(W, I, M), nmf, K, make_spec(I, J, M, X));
  });
}

}  // extern "C"
