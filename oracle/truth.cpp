// truth.cpp -- extended-precision GROUND TRUTH for the parity tests (test
// infrastructure only; nothing in paper_1908_01964_b200/ links or loads it).
//
// The double-precision oracle (rcscm_oracle.cpp) and the CUDA path both round
// at every step; on slots where an update cancels (r_u = (g rho_aa q + rho_xx
// - 2 g Re(.))/M with terms ~1e8 x the result, solver_accel.hpp:160-176), or
// where the naive rule inverts a nearly rank-one R_x (solver_naive.hpp:186-197),
// the two disagree by more than 1e-9 and neither comparison says which is
// right. This file evaluates the SAME formulas on the SAME double inputs (each
// taken as an exact value) in IEEE binary128 (__float128: 113-bit significand,
// ~1e-34), so every rounding error of a double implementation shows up against
// it, and only the final result is rounded to double:
//
//   truth_accel_one_iter  Algorithm 2, one iteration from params0:
//                         precompute_sigma/tau solver_accel.hpp:33-64 (full
//                         x^H (R'^+ x) form), rho_second_stage :113-129,
//                         compute_gamma :67-76, update_rh :134-141,
//                         update_lambda :143-158, update_ru :160-176.
//   truth_naive_one_iter  the naive rule, one iteration: naive_e_step_bin_impl
//                         solver_naive.hpp:153-246 (R_x lower triangle + Hermitian
//                         mirror, exact inverse by Gauss-Jordan with partial
//                         pivoting in binary128), naive_iteration_bin_impl
//                         :319-386 (r_h, lambda from b^H hat b / r~_u, R_u^-1,
//                         r_u = Re tr(R_u^-1 hat)/M).
//   truth_wiener          extract_target wiener.hpp:19-43 (dry only) from given
//                         params, in binary128.
//
// Both one-iteration functions also return a first-order ROUNDING SCALE per
// output, B_rh, B_ru (per slot) and B_lam (per bin): the standard a-priori
// forward-error bound of a double evaluation of the same formulas (Higham,
// "Accuracy and Stability of Numerical Algorithms", ch. 3: a computed sum or
// dot product errs by at most ~n eps times the sum of the magnitudes of its
// terms), propagated through every step -- for Algorithm 2 the magnitudes of
// the precompute dot products, of the rho / gamma / residual terms and of the
// three terms of the r_u update, which cancel when r_u is small; for the naive
// rule additionally the 1-norm condition numbers kappa(R_x), kappa(R_u) of the
// matrices it inverts. Any double implementation of the formulas, in any
// operation order, is expected within C eps B of the truth for a modest C;
// tests/test_truth.py measures C for the oracle (the reference's arithmetic)
// and tests/test_gpu_truth.py holds the GPU to the same C.
//
// Floors are std::max(v, eps) as in the reference. Layouts are the oracle's
// (rcscm_oracle.h): X [i][t][m]; a, b [i][m]; R', R'^+ [i] M x M col-major;
// r_h, r_u, dry element (i, t) at i + t*I.
#include <algorithm>
#include <cstdint>
#include <thread>
#include <vector>

namespace {

typedef __float128 Q;

struct C {
  Q re, im;
};
inline C mk(Q r, Q i) { return C{r, i}; }
inline C add(C a, C b) { return C{a.re + b.re, a.im + b.im}; }
inline C sub(C a, C b) { return C{a.re - b.re, a.im - b.im}; }
inline C mul(C a, C b) { return C{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
inline C conj(C a) { return C{a.re, -a.im}; }
inline C scal(C a, Q s) { return C{a.re * s, a.im * s}; }
inline Q norm(C a) { return a.re * a.re + a.im * a.im; }
inline Q qabs(Q v) { return v < 0 ? -v : v; }
inline C cdiv(C a, C b) {
  const Q d = norm(b);
  return C{(a.re * b.re + a.im * b.im) / d, (a.im * b.re - a.re * b.im) / d};
}
inline C ld(const double* p, int64_t k) { return C{p[2 * k], p[2 * k + 1]}; }
inline Q qmax(Q v, Q lo) { return v < lo ? lo : v; }  // std::max(v, lo)
// |z| for the rounding scales (only magnitudes: the double sqrt is plenty)
inline Q sqrtq_(Q v) { return static_cast<Q>(__builtin_sqrt(static_cast<double>(v))); }

// Run f(i) for bins [0, I) on all host threads (bins are independent).
template <class F>
void for_bins(int64_t I, F f) {
  const int nt = std::max(1u, std::thread::hardware_concurrency());
  std::vector<std::thread> th;
  for (int k = 0; k < nt; ++k)
    th.emplace_back([&, k] {
      for (int64_t i = k; i < I; i += nt) f(i);
    });
  for (auto& t : th) t.join();
}

// Inverse of a general M x M complex matrix (col-major) by Gauss-Jordan with
// partial pivoting; false if singular.
bool inverse(int M, std::vector<C> A, std::vector<C>* out) {
  std::vector<C>& R = *out;
  R.assign(M * M, mk(0, 0));
  for (int k = 0; k < M; ++k) R[k + k * M] = mk(1, 0);
  for (int c = 0; c < M; ++c) {
    int p = c;
    for (int r = c + 1; r < M; ++r)
      if (norm(A[r + c * M]) > norm(A[p + c * M])) p = r;
    if (norm(A[p + c * M]) == 0) return false;
    if (p != c)
      for (int k = 0; k < M; ++k) {
        std::swap(A[c + k * M], A[p + k * M]);
        std::swap(R[c + k * M], R[p + k * M]);
      }
    const C piv = A[c + c * M];
    for (int k = 0; k < M; ++k) {
      A[c + k * M] = cdiv(A[c + k * M], piv);
      R[c + k * M] = cdiv(R[c + k * M], piv);
    }
    for (int r = 0; r < M; ++r) {
      if (r == c) continue;
      const C f = A[r + c * M];
      for (int k = 0; k < M; ++k) {
        A[r + k * M] = sub(A[r + k * M], mul(f, A[c + k * M]));
        R[r + k * M] = sub(R[r + k * M], mul(f, R[c + k * M]));
      }
    }
  }
  return true;
}

}  // namespace

extern "C" {

int truth_accel_one_iter(int64_t I, int64_t J, int M, const double* a, const double* Rpp, const double* b,
                         const double* r_h0, const double* r_u0, const double* lambda0, double alpha, double beta,
                         double eps, const double* X, double* r_h, double* r_u, double* lambda, double* B_rh,
                         double* B_ru, double* B_lam) {
  for_bins(I, [&](int64_t i) {
    std::vector<C> av(M), bv(M), P(M * M), pa(M);
    std::vector<Q> pa_abs(M, 0);
    for (int m = 0; m < M; ++m) {
      av[m] = ld(a, i * M + m);
      bv[m] = ld(b, i * M + m);
    }
    for (int k = 0; k < M * M; ++k) P[k] = ld(Rpp, i * M * M + k);
    // precompute_sigma / precompute_tau (solver_accel.hpp:33-64)
    C sab = mk(0, 0);
    for (int m = 0; m < M; ++m) sab = add(sab, mul(conj(av[m]), bv[m]));
    for (int r = 0; r < M; ++r) {
      C s = mk(0, 0);
      for (int c = 0; c < M; ++c) {
        s = add(s, mul(P[r + c * M], av[c]));
        pa_abs[r] += sqrtq_(norm(P[r + c * M])) * sqrtq_(norm(av[c]));
      }
      pa[r] = s;
    }
    C aa = mk(0, 0);
    Q sab_abs = 0, taa_abs = 0;
    for (int m = 0; m < M; ++m) {
      aa = add(aa, mul(conj(av[m]), pa[m]));
      sab_abs += sqrtq_(norm(av[m])) * sqrtq_(norm(bv[m]));
      taa_abs += sqrtq_(norm(av[m])) * pa_abs[m];
    }
    const Q taa = qmax(aa.re, 0);
    const Q lam0 = lambda0[i];
    const Q ab2 = norm(sab);
    const Q trho_aa = taa + ab2 / lam0;
    const Q trho_aa_abs = taa_abs + sab_abs * sab_abs / lam0;
    std::vector<C> sbx(J), tax(J), trax(J);
    std::vector<Q> txx(J), g(J), g_abs(J), sbx_abs(J), tax_abs(J), txx_abs(J), trax_abs(J);
    Q acc = 0, acc_abs = 0;
    for (int64_t t = 0; t < J; ++t) {
      std::vector<C> x(M);
      for (int m = 0; m < M; ++m) x[m] = ld(X, (i * J + t) * M + m);
      C s1 = mk(0, 0), s2 = mk(0, 0), s3 = mk(0, 0);
      Q a1 = 0, a2 = 0, a3 = 0;
      for (int m = 0; m < M; ++m) {
        s1 = add(s1, mul(conj(bv[m]), x[m]));
        s2 = add(s2, mul(conj(pa[m]), x[m]));
        a1 += sqrtq_(norm(bv[m])) * sqrtq_(norm(x[m]));
        a2 += pa_abs[m] * sqrtq_(norm(x[m]));
      }
      for (int r = 0; r < M; ++r) {
        C px = mk(0, 0);
        for (int c = 0; c < M; ++c) {
          px = add(px, mul(P[r + c * M], x[c]));
          a3 += sqrtq_(norm(x[r])) * sqrtq_(norm(P[r + c * M])) * sqrtq_(norm(x[c]));
        }
        s3 = add(s3, mul(conj(x[r]), px));
      }
      sbx_abs[t] = a1;
      tax_abs[t] = a2;
      txx_abs[t] = a3;
      sbx[t] = s1;
      tax[t] = s2;
      txx[t] = qmax(s3.re, 0);
      // rho~ with lambda0, gamma (solver_accel.hpp:67-76, :113-129)
      trax[t] = add(tax[t], scal(mul(sab, sbx[t]), 1 / lam0));
      trax_abs[t] = tax_abs[t] + sab_abs * sbx_abs[t] / lam0;
      const Q rh = r_h0[i + t * I], ru = r_u0[i + t * I];
      const Q D = ru + rh * trho_aa;
      g[t] = rh / D;
      g_abs[t] = g[t] * (1 + rh * trho_aa_abs / D);  // error(gamma) <~ eps g_abs
      // update_rh (:134-141)
      const Q vh = (g[t] * (ru + g[t] * norm(trax[t])) + beta) / (alpha + 2);
      r_h[i + t * I] = static_cast<double>(qmax(vh, eps));
      if (B_rh)
        B_rh[i + t * I] = static_cast<double>(
            (g_abs[t] * ru + 3 * g_abs[t] * g[t] * trax_abs[t] * trax_abs[t] + beta) / (alpha + 2));
      // update_lambda (:143-158)
      const C resid = sub(sbx[t], mul(scal(conj(sab), g[t]), trax[t]));
      const Q term = g[t] * ab2 + norm(resid) / ru;
      const Q resid_abs = sbx_abs[t] + g_abs[t] * sab_abs * trax_abs[t];
      acc += term;
      acc_abs += g_abs[t] * sab_abs * sab_abs + resid_abs * resid_abs / ru;
    }
    const Q lam = qmax(acc / static_cast<Q>(J), eps);
    lambda[i] = static_cast<double>(lam);
    const Q lam_abs = acc_abs / static_cast<Q>(J);
    if (B_lam) B_lam[i] = static_cast<double>(lam_abs);
    const Q fl = 1 + lam_abs / lam;  // 1/lambda's relative error carries into every rho
    // rho with the new lambda, update_ru (:160-176)
    const Q rho_aa = taa + ab2 / lam;
    for (int64_t t = 0; t < J; ++t) {
      const C rho_ax = add(tax[t], scal(mul(sab, sbx[t]), 1 / lam));
      const Q rho_xx = txx[t] + norm(sbx[t]) / lam;
      const Q ru = r_u0[i + t * I];
      const Q t1 = g[t] * rho_aa * (ru + g[t] * norm(trax[t]));
      const Q t3 = 2 * g[t] * mul(trax[t], conj(rho_ax)).re;
      const Q val = (t1 + rho_xx - t3) / static_cast<Q>(M);
      r_u[i + t * I] = static_cast<double>(qmax(val, eps));
      if (B_ru) {
        const Q raa_abs = taa_abs + sab_abs * sab_abs / lam * fl;
        const Q rax_abs = tax_abs[t] + sab_abs * sbx_abs[t] / lam * fl;
        const Q rxx_abs = txx_abs[t] + sbx_abs[t] * sbx_abs[t] / lam * fl;
        const Q t1_abs = g_abs[t] * raa_abs * (ru + 3 * g[t] * trax_abs[t] * trax_abs[t]);
        const Q t3_abs = 2 * g_abs[t] * trax_abs[t] * rax_abs;
        B_ru[i + t * I] = static_cast<double>((t1_abs + rxx_abs + t3_abs) / static_cast<Q>(M));
      }
    }
  });
  return 0;
}

int truth_naive_one_iter(int64_t I, int64_t J, int M, const double* a, const double* Rp, const double* b,
                         const double* r_h0, const double* r_u0, const double* lambda0, double alpha, double beta,
                         double eps, const double* X, double* r_h, double* r_u, double* lambda, double* B_rh,
                         double* B_ru, double* B_lam) {
  int bad = 0;
  auto cabs = [](C z) { return sqrtq_(norm(z)); };
  auto norm1 = [&](const std::vector<C>& A) {  // max column sum of |a_rc|
    Q best = 0;
    for (int c = 0; c < M; ++c) {
      Q s = 0;
      for (int r = 0; r < M; ++r) s += cabs(A[r + c * M]);
      best = std::max(best, s);
    }
    return best;
  };
  auto vnorm1 = [&](const std::vector<C>& v) {
    Q s = 0;
    for (const C& z : v) s += cabs(z);
    return s;
  };
  for_bins(I, [&](int64_t i) {
    std::vector<C> av(M), bv(M), Rt(M * M), Rx(M * M), Rxi, Ru(M * M), Rui;
    for (int m = 0; m < M; ++m) {
      av[m] = ld(a, i * M + m);
      bv[m] = ld(b, i * M + m);
    }
    const Q a1 = vnorm1(av), b1 = vnorm1(bv);
    const Q lam0 = lambda0[i];
    for (int c = 0; c < M; ++c)
      for (int r = 0; r < M; ++r)
        Rt[r + c * M] = add(ld(Rp, i * M * M + r + c * M), scal(mul(bv[r], conj(bv[c])), lam0));
    const Q nRt = norm1(Rt);
    std::vector<std::vector<C>> hat(J, std::vector<C>(M * M));
    std::vector<Q> H_abs(J), nHat(J);
    Q lam_acc = 0, lam_abs = 0;
    for (int64_t t = 0; t < J; ++t) {
      const Q rh = r_h0[i + t * I], ru = r_u0[i + t * I];
      std::vector<C> x(M);
      for (int m = 0; m < M; ++m) x[m] = ld(X, (i * J + t) * M + m);
      const Q x1 = vnorm1(x);
      // R_x = rh a a^H + ru R~_u (lower triangle, Hermitian mirror; :186-191)
      for (int c = 0; c < M; ++c) {
        for (int r = c; r < M; ++r) Rx[r + c * M] = add(mul(av[r], scal(conj(av[c]), rh)), scal(Rt[r + c * M], ru));
        for (int r = 0; r < c; ++r) Rx[r + c * M] = conj(Rx[c + r * M]);
      }
      if (!inverse(M, Rx, &Rxi)) {
        bad = 1;
        return;
      }
      const Q nRi = norm1(Rxi), kx = norm1(Rx) * nRi;  // 1-norm condition number of R_x
      Q a_rxi_a = 0;
      C x_rxi_a = mk(0, 0);
      for (int r = 0; r < M; ++r) {
        C s = mk(0, 0);
        for (int c = 0; c < M; ++c) s = add(s, mul(Rxi[r + c * M], av[c]));
        a_rxi_a += mul(conj(av[r]), s).re;
        x_rxi_a = add(x_rxi_a, mul(conj(x[r]), s));
      }
      const Q hrh = rh - rh * rh * a_rxi_a + norm(scal(x_rxi_a, rh));
      r_h[i + t * I] = static_cast<double>(qmax((hrh + beta) / (alpha + 2), eps));
      const Q xa = cabs(x_rxi_a);
      if (B_rh)
        B_rh[i + t * I] = static_cast<double>(
            (rh + rh * rh * (qabs(a_rxi_a) + a1 * a1 * kx * nRi) + rh * rh * (xa * xa + 2 * xa * x1 * a1 * kx * nRi) +
             beta) / (alpha + 2));
      std::vector<C> RR(M * M), v(M);
      for (int r = 0; r < M; ++r) {
        C vx = mk(0, 0);
        for (int c = 0; c < M; ++c) {
          C s = mk(0, 0);
          for (int k = 0; k < M; ++k) s = add(s, mul(Rt[r + k * M], Rxi[k + c * M]));
          RR[r + c * M] = s;
          vx = add(vx, mul(s, x[c]));
        }
        v[r] = vx;
      }
      std::vector<C>& H = hat[t];
      for (int c = 0; c < M; ++c) {
        for (int r = c; r < M; ++r) {
          C s = mk(0, 0);
          for (int k = 0; k < M; ++k) s = add(s, mul(RR[r + k * M], Rt[k + c * M]));
          H[r + c * M] = add(sub(scal(Rt[r + c * M], ru), scal(s, ru * ru)), scal(mul(v[r], conj(v[c])), ru * ru));
        }
        for (int r = 0; r < c; ++r) H[r + c * M] = conj(H[c + r * M]);
      }
      const Q v1 = vnorm1(v);
      // rounding scale of hat R_u: r_u R~_u, r_u^2 R~_u R_x^-1 R~_u (inverse error
      // ~ eps kappa(R_x) ||R_x^-1||) and r_u^2 v v^H (v = R~_u R_x^-1 x likewise)
      H_abs[t] = ru * nRt + ru * ru * nRt * nRt * nRi * kx + ru * ru * (v1 * v1 + 2 * v1 * nRt * kx * nRi * x1);
      nHat[t] = norm1(H);
      C q = mk(0, 0);  // b^H hat b
      for (int r = 0; r < M; ++r) {
        C s = mk(0, 0);
        for (int c = 0; c < M; ++c) s = add(s, mul(H[r + c * M], bv[c]));
        q = add(q, mul(conj(bv[r]), s));
      }
      lam_acc += q.re / ru;
      lam_abs += b1 * b1 * H_abs[t] / ru;
    }
    const Q lam = qmax(lam_acc / static_cast<Q>(J), eps);
    lambda[i] = static_cast<double>(lam);
    lam_abs /= static_cast<Q>(J);
    if (B_lam) B_lam[i] = static_cast<double>(lam_abs);
    for (int c = 0; c < M; ++c)
      for (int r = 0; r < M; ++r)
        Ru[r + c * M] = add(ld(Rp, i * M * M + r + c * M), scal(mul(bv[r], conj(bv[c])), lam));
    if (!inverse(M, Ru, &Rui)) {
      bad = 1;
      return;
    }
    const Q nRui = norm1(Rui), ku = norm1(Ru) * nRui;
    for (int64_t t = 0; t < J; ++t) {
      Q tr = 0;
      for (int r = 0; r < M; ++r)
        for (int k = 0; k < M; ++k) tr += mul(Rui[r + k * M], hat[t][k + r * M]).re;
      r_u[i + t * I] = static_cast<double>(qmax(tr / static_cast<Q>(M), eps));
      // tr(R_u^-1 hat)/M: hat's rounding, R_u^-1's (kappa(R_u)) and lambda's through R_u
      if (B_ru)
        B_ru[i + t * I] =
            static_cast<double>(nRui * H_abs[t] + ku * nRui * nHat[t] + nRui * nRui * b1 * b1 * lam_abs * nHat[t]);
    }
  });
  return bad ? 3 : 0;
}

int truth_wiener(int64_t I, int64_t J, int M, const double* a, const double* Rpp, const double* b, const double* r_h,
                 const double* r_u, const double* lambda, const double* X, double* dry) {
  for_bins(I, [&](int64_t i) {
    std::vector<C> av(M), bv(M), P(M * M), pa(M);
    for (int m = 0; m < M; ++m) {
      av[m] = ld(a, i * M + m);
      bv[m] = ld(b, i * M + m);
    }
    for (int k = 0; k < M * M; ++k) P[k] = ld(Rpp, i * M * M + k);
    C sab = mk(0, 0);
    for (int m = 0; m < M; ++m) sab = add(sab, mul(conj(av[m]), bv[m]));
    for (int r = 0; r < M; ++r) {
      C s = mk(0, 0);
      for (int c = 0; c < M; ++c) s = add(s, mul(P[r + c * M], av[c]));
      pa[r] = s;
    }
    C aa = mk(0, 0);
    for (int m = 0; m < M; ++m) aa = add(aa, mul(conj(av[m]), pa[m]));
    const Q lam = lambda[i];
    const Q rho_aa = qmax(aa.re, 0) + norm(sab) / lam;
    for (int64_t t = 0; t < J; ++t) {
      C sbx = mk(0, 0), tax = mk(0, 0);
      for (int m = 0; m < M; ++m) {
        const C x = ld(X, (i * J + t) * M + m);
        sbx = add(sbx, mul(conj(bv[m]), x));
        tax = add(tax, mul(conj(pa[m]), x));
      }
      const C rho_ax = add(tax, scal(mul(sab, sbx), 1 / lam));
      const Q rh = r_h[i + t * I], ru = r_u[i + t * I];
      const Q g = rh / (ru + rh * rho_aa);
      const C s = scal(rho_ax, g);
      dry[2 * (i + t * I)] = static_cast<double>(s.re);
      dry[2 * (i + t * I) + 1] = static_cast<double>(s.im);
    }
  });
  return 0;
}

}  // extern "C"
