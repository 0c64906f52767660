/*
 * rcscm_oracle.h -- C ABI of the CPU ORACLE (test infrastructure only).
 *
 * The oracle is a plain C++17 restatement of the reference's hot path
 * (/root/reference/proj/include/rcscm/{linalg,model,solver_accel,solver_naive,
 * wiener,verify}.hpp). It exists so that tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py can CHECK the CUDA product
 * path. Nothing in paper_1908_01964_b200/ links, loads or calls it.
 *
 * Layouts are the reference's own (Eigen column-major, complex128 interleaved):
 *   X, image, noise : [i][t][m]            (Spectrogram::bins[i] is M x J col-major)
 *   a, b            : [i][m]
 *   Rp, Rpp, W, A   : [i][r + c*M]          (M x M col-major per bin)
 *   r_h, r_u, gamma,
 *   sigma_bx, tau_ax,
 *   tau_xx, dry     : element (i, t) at i + t*I   (Eigen MatR/MatC I x J)
 *   T (I x K)       : i + k*I ;  V (K x J) : k + t*K
 * Complex arrays are passed as double* with (re, im) pairs.
 *
 * Return codes follow the reference's exception split (types.hpp:20-30):
 *   0 ok, 2 InvalidInputError, 3 NumericalError; message via oracle_last_error().
 */
#ifndef RCSCM_ORACLE_H
#define RCSCM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* oracle_last_error(void);

/* linalg.hpp:25-117 */
int oracle_hermitian_eig(int M, const double* H, double* values, double* vectors);
int oracle_pseudo_inverse_psd(int M, const double* H, double rank_tol, double* out);
int oracle_null_eigenvector(int M, const double* H, double rank_tol, double* out);
int oracle_normalize_phase(int M, const double* v, double* out);
int oracle_sherman_morrison_inverse(int M, const double* Rinv, const double* a,
                                    double c, double d, double* out);
int oracle_rank_one_restored_inverse(int M, const double* Rpp, const double* b,
                                     double lambda, double* out);

/* model.hpp:58-90 build_noise_scm */
int oracle_build_noise_scm(int64_t I, int64_t J, int M, const double* X,
                           const double* W, const double* A, int n_h,
                           double rank_tol, double* a, double* Rp, double* Rpp,
                           double* b);
/* model.hpp:95-124 init_params (T, V are NmfModel::T[n_h], V[n_h]) */
int oracle_init_params(int64_t I, int64_t J, int M, int K, const double* X,
                       const double* W, const double* A, int n_h,
                       const double* Rp, const double* Rpp, const double* T,
                       const double* V, double* r_h, double* r_u, double* lambda);
/* model.hpp:129-157 map_objective */
int oracle_map_objective(int64_t I, int64_t J, int M, const double* a,
                         const double* Rp, const double* b, const double* r_h,
                         const double* r_u, const double* lambda, double alpha,
                         double beta, const double* X, double* out);

/* solver_accel.hpp:33-64 precompute_sigma / precompute_tau */
int oracle_precompute(int64_t I, int64_t J, int M, const double* a,
                      const double* Rpp, const double* b, const double* X,
                      double* sigma_ab, double* sigma_bx, double* tau_aa,
                      double* tau_ax, double* tau_xx);
/* solver_accel.hpp:67-76 */
int oracle_compute_gamma(int64_t I, int64_t J, const double* r_h, const double* r_u,
                         const double* trho_aa, double* gamma);
/* solver_accel.hpp:80-109 (rho_xx may be NULL) */
int oracle_rho_first_stage(int64_t I, int64_t J, int M, const double* Rp,
                           const double* a, const double* b, const double* X,
                           const double* lambda, double* rho_aa, double* rho_ax,
                           double* rho_xx);
/* solver_accel.hpp:113-129 (rho_xx may be NULL) */
int oracle_rho_second_stage(int64_t I, int64_t J, const double* sigma_ab,
                            const double* sigma_bx, const double* tau_aa,
                            const double* tau_ax, const double* tau_xx,
                            const double* lambda, double* rho_aa, double* rho_ax,
                            double* rho_xx);
/* solver_accel.hpp:134-176 */
int oracle_update_rh(int64_t I, int64_t J, const double* gamma, const double* r_u,
                     const double* trho_ax, double alpha, double beta, double eps,
                     double* r_h_out);
int oracle_update_lambda(int64_t I, int64_t J, const double* gamma,
                         const double* r_u, const double* sigma_ab,
                         const double* sigma_bx, const double* trho_ax, double eps,
                         double* lambda_out);
int oracle_update_ru(int64_t I, int64_t J, int M, const double* gamma,
                     const double* r_u, const double* rho_aa, const double* rho_ax,
                     const double* trho_ax, const double* rho_xx, double eps,
                     double* r_u_out);

/* solver_naive.hpp:46-146 closed-form Hermitian PD inverse (S = 2, 3, 4) and
 * the LLT path used for other sizes. Returns 3 when not PD. */
int oracle_hermitian_pd_inverse(int M, const double* R, double* out);
/* solver_naive.hpp:267-279 e_step: hat_r_h I x J col-major, hat_R_u [i][t][M*M] */
int oracle_e_step(int64_t I, int64_t J, int M, const double* a, const double* Rp,
                  const double* b, const double* r_h, const double* r_u,
                  const double* lambda, const double* X, double* hat_r_h,
                  double* hat_R_u);
/* solver_naive.hpp:282-311 m_step */
int oracle_m_step(int64_t I, int64_t J, int M, const double* hat_r_h,
                  const double* hat_R_u, const double* Rp, const double* b,
                  const double* r_u_old, double alpha, double beta, double eps,
                  double* r_h, double* r_u, double* lambda);

typedef struct {
  int iters;
  int compute_objective;
  int record_trajectory;
  double rel_obj_tol;
  int threads;
  double eps_var;
  double gamma_fault;
} oracle_solver_opts;

/* backend: 0 = run_naive (solver_naive.hpp:412), 1 = run_algorithm1
 * (solver_accel.hpp:246), 2 = run_algorithm2 (solver_accel.hpp:254).
 * Outputs: r_h/r_u/lambda (final params). Optional (may be NULL):
 * objective[iters+1], iter_seconds[iters], traj_r_h/traj_r_u [iters][I*J],
 * traj_lambda [iters][I]. n_obj / n_iter receive the counts written. */
int oracle_run(int backend, int64_t I, int64_t J, int M, const double* a,
               const double* Rp, const double* Rpp, const double* b,
               const double* r_h0, const double* r_u0, const double* lambda0,
               double alpha, double beta, const double* X,
               const oracle_solver_opts* opt, double* r_h, double* r_u,
               double* lambda, double* objective, int* n_obj,
               double* iter_seconds, int* n_iter, double* traj_r_h,
               double* traj_r_u, double* traj_lambda);

/* wiener.hpp:19-43 / :46-53 (image/noise may be NULL) */
int oracle_extract_target(int64_t I, int64_t J, int M, const double* a,
                          const double* Rpp, const double* b, const double* r_h,
                          const double* r_u, const double* lambda, const double* X,
                          double* image, double* dry);
int oracle_extract_noise(int64_t I, int64_t J, int M, const double* a,
                         const double* Rpp, const double* b, const double* r_h,
                         const double* r_u, const double* lambda, const double* X,
                         double* noise);

/* verify.hpp:22-56 make_verify_instance (mt19937_64 + normal_distribution) */
int oracle_make_verify_instance(int64_t I, int64_t J, int M, uint64_t seed,
                                double* X, double* a, double* Rp, double* Rpp,
                                double* b, double* r_h, double* r_u,
                                double* lambda);
/* verify.hpp:60-68 */
double oracle_trajectory_distance(int64_t I, int64_t J, const double* r_h_a,
                                  const double* r_u_a, const double* lam_a,
                                  const double* r_h_b, const double* r_u_b,
                                  const double* lam_b);

/* ilrma.hpp:53-73 sphere (Q: [i][M*M] col-major, Xw: [i][t][m]) */
int oracle_sphere(int64_t I, int64_t J, int M, const double* X, double* Q, double* Xw);
/* ilrma.hpp:145-240 run_ilrma (W, A: [i][M*M]; T: [n][I x K]; V: [n][K x J], col-major) */
int oracle_run_ilrma(int64_t I, int64_t J, int M, int K, int iters, uint64_t seed, const double* X, double* W,
                     double* A, double* T, double* V);
/* ilrma.hpp:86-98 ilrma_objective */
int oracle_ilrma_objective(int64_t I, int64_t J, int M, int K, const double* X, const double* W, const double* T,
                           const double* V, double* out);

#ifdef __cplusplus
}
#endif
#endif /* RCSCM_ORACLE_H */
