/* SPDX-License-Identifier: MIT
 * TEST INFRASTRUCTURE ONLY — C-ABI of the CPU parity oracle (liboracle.so),
 * bound by tests/ through ctypes (oracle/oracle.py). Never linked by the
 * product library.
 *
 * The flat problem layout (orc_problem_view) is byte-compatible with the
 * product's scenopt_problem_view (include/scenopt_b200.h) so one set of
 * numpy arrays feeds both sides of every parity test.
 */
#ifndef SCENOPT_ORACLE_CAPI_H
#define SCENOPT_ORACLE_CAPI_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_problem_view {
  int32_t nx, nu, num_stages, num_nodes;
  const int32_t* ancestor;      /* [n], -1 at the root */
  const double* probability;    /* [n] */
  const int32_t* stage_offsets; /* [num_stages + 2] */
  const double* root_state;     /* [nx] */
  const double *A, *B, *c;      /* [n][nx*nx], [n][nx*nu], [n][nx], column-major, slot 0 unused */
  const double *Q, *R, *S;      /* [n][nx*nx], [n][nu*nu], [n][nu*nx] */
  const double *q, *r;          /* [n][nx], [n][nu] */
  const int32_t* stage_rows;    /* [n], m_i (0 at the root) */
  const double *F, *G;          /* stage rows in dual order: node i block at dual_offset[i]*nx / *nu */
  const int32_t* g_kind;        /* [n] 0 none, 1 box, 2 scaled_l1 */
  const double* g_gamma;        /* [n] */
  const double *P, *p;          /* [L][nx*nx], [L][nx] */
  const int32_t* terminal_rows; /* [L] */
  const double* FN;             /* terminal rows: leaf l block at (tdual_offset[l]-S)*nx */
  const int32_t* tg_kind;       /* [L] */
  const double* tg_gamma;       /* [L] */
  const double *zmin, *zmax;    /* [dual_dim], dual layout (box rows only meaningful) */
} orc_problem_view;

typedef struct orc_solver_config {
  double lambda0, eps, eps_curv, eps_bt, beta_bt;
  int32_t memory, max_iters, backtracking_rule, warm_start, warm_start_iters, precondition,
      nama_parallel_linesearch, nama_update_tlambda;
} orc_solver_config;

typedef struct orc_report_summary {
  int32_t status, iterations, verified, trace_len;
  uint64_t dual_grad_calls, hessian_vec_calls, prox_calls, conj_calls, lipschitz_calls;
  double lipschitz_estimate, lambda_final, eps, residual_inf, wall_ms, verify_residual_inf,
      verify_subdiff_dist;
} orc_report_summary;

typedef struct orc_instance_options {
  int32_t with_box, with_l1, with_none, affine, stage_rows_lo, stage_rows_hi, feasible_boxes;
} orc_instance_options;

typedef struct orc_problem orc_problem;
typedef struct orc_factor orc_factor;
typedef struct orc_g orc_g;
typedef struct orc_rng orc_rng;
typedef struct orc_lbfgs orc_lbfgs;
typedef struct orc_report orc_report;

const char* orc_last_error(void);

/* problems */
int orc_problem_from_view(const orc_problem_view* v, orc_problem** out);
int orc_problem_view_get(orc_problem* p, orc_problem_view* v, int32_t* dual_dim);
void orc_problem_free(orc_problem* p);
int orc_gen_random(uint64_t seed, int nx, int nu, int horizon, const int32_t* branching, int nbr,
                   orc_problem** out);
/* generators.hpp:39-234 (spring-mass benchmark). Arrays of length 0 take the defaults;
 * transition is row-major [transition_rows x transition_cols]. */
typedef struct orc_spring_mass_params {
  double mass_kg, stiffness, damping, input_bound, velocity_bound;
  int32_t horizon;
  double sampling, state_weight, input_weight, terminal_weight;
  int32_t initial_len, transition_rows, transition_cols, mode_values_len, root_state_len;
  const double* initial_probs;
  const double* transition;
  const double* mode_values;
  const double* root_state;
} orc_spring_mass_params;
int orc_gen_spring_mass(int masses, const orc_spring_mass_params* par, orc_problem** out);
/* series exponential (test_generators.cpp:23-38), column-major n x n */
int orc_expm_series(const double* X, int n, double* out);
int orc_spring_mass_continuous(int masses, const orc_spring_mass_params* par, double* A, double* B);
/* `count` consecutive sample_initial_state draws from mt19937_64(seed) */
int orc_sample_initial_states(int masses, const orc_spring_mass_params* par, uint64_t seed, int count,
                              double* out);
int orc_problem_validate(const orc_problem* p, char* buf, int buflen);
int orc_problem_layout(const orc_problem* p, int32_t* dual_offset, int32_t* tdual_offset);
int orc_precondition(const orc_problem* p, orc_problem** out);
int orc_probability_roots(const orc_problem* p, double* out);

/* rng + test-support generators */
int orc_rng_new(uint64_t seed, orc_rng** out);
void orc_rng_free(orc_rng* r);
double orc_rng_uniform(orc_rng* r, double lo, double hi);
int orc_rng_integer(orc_rng* r, int lo, int hi);
void orc_rng_vector(orc_rng* r, int n, double scale, double* out);
void orc_rng_matrix(orc_rng* r, int rows, int cols, double scale, double* out);
int orc_random_instance(orc_rng* r, int stages, int max_nodes, int nx, int nu,
                        const orc_instance_options* opt, orc_problem** out);
int orc_markov_instance(orc_rng* r, const double* transition, const double* initial, int modes,
                        int horizon, int nx, int nu, const orc_instance_options* opt,
                        orc_problem** out);
int orc_tree_from_markov(const double* transition, const double* initial, int modes, int horizon,
                         int32_t* num_nodes, int32_t* ancestor, double* probability,
                         int32_t* stage_offsets, int32_t* mode, int cap);

/* factor */
int orc_factor_create(const orc_problem* p, orc_factor** out);
void orc_factor_free(orc_factor* f);
int orc_refactor_affine(orc_factor* f, const orc_problem* p);
/* flat export: gain [F][nu*nx], child_to_input [n][nu*nx], closed_loop [n][nx*nx],
 * dual_to_input/dual_to_costate concatenated by child_dual_offset (nu*M, nx*M),
 * input_affine [F][nu], costate_affine [F][nx], value_quad [n][nx*nx], leaf_costate_affine [L][nx] */
int orc_factor_export(const orc_factor* f, double* gain, double* child_to_input, double* closed_loop,
                      double* dual_to_input, double* dual_to_costate, double* input_affine,
                      double* costate_affine, double* value_quad, double* leaf_costate_affine);

/* oracles */
int orc_sweep(const orc_factor* f, const orc_problem* p, const double* y, int affine, double* x,
              double* u);
int orc_apply_H(const orc_problem* p, const double* x, const double* u, double* z);
int orc_apply_H_adjoint(const orc_problem* p, const double* y, double* x, double* u);
int orc_eval_f(const orc_problem* p, const double* x, const double* u, double* out);
int orc_fhat_value(const orc_factor* f, const orc_problem* p, const double* y, double* out);

/* nonsmooth */
int orc_g_from_problem(const orc_problem* p, orc_g** out);
int orc_g_create(int dim, int nblocks, const int32_t* offset, const int32_t* size,
                 const double* weight, const int32_t* kind, const double* gamma,
                 const double* zmin, const double* zmax, orc_g** out);
void orc_g_free(orc_g* g);
int orc_prox_g(const orc_g* g, const double* v, double gamma_prox, double* out);
int orc_conj_value_g(const orc_g* g, const double* w, double* out);
int orc_prox_g_conj(const orc_g* g, const double* v, double lambda, double* out);
int orc_dist_subdiff_inf(const orc_g* g, const double* y, const double* z, double* out);

/* forward-backward machinery: outputs are caller-owned dual/primal buffers,
 * scalars = {fhat, conj_T, znorm_sq, value} */
int orc_fb_step(const orc_factor* f, const orc_problem* p, const orc_g* g, const double* y,
                double lambda, double* x, double* u, double* Hx, double* z, double* R, double* T,
                double* scalars);
int orc_fbe_grad(const orc_factor* f, const orc_problem* p, const double* R, double lambda,
                 double* grad);
/* certificate: plain (shift == NULL) or shifted (NAMA). Takes the fb state
 * (y, Hx, lambda, scalars) and evaluates taus[k]; out per tau: delta, and
 * optionally w/Hx_w/z/R/T of the LAST tau into the given buffers.
 * cert_scalars = {alpha1, alpha2, conj_anchor, znorm_sq_anchor, value_anchor, fhat_anchor} */
int orc_linesearch_cert(const orc_factor* f, const orc_problem* p, const orc_g* g,
                        const double* y, const double* Hx, double lambda, const double* state_scalars,
                        const double* shift, const double* dir, int ntau, const double* taus,
                        double* deltas, double* cert_scalars, double* cert_fhat, double* w,
                        double* Hx_w, double* z, double* R, double* T);

/* L-BFGS */
int orc_lbfgs_new(int memory, double eps_curv, orc_lbfgs** out);
void orc_lbfgs_free(orc_lbfgs* b);
int orc_lbfgs_push(orc_lbfgs* b, int n, const double* step, const double* change, double scale_ref);
int orc_lbfgs_apply(const orc_lbfgs* b, int n, const double* grad, double* out);
void orc_lbfgs_clear(orc_lbfgs* b);
int orc_lbfgs_size(const orc_lbfgs* b);
double orc_lbfgs_gamma0(const orc_lbfgs* b);

/* solvers: kind 0 MINFBE, 1 NAMA, 2 GPAD */
int orc_estimate_lipschitz(const orc_factor* f, const orc_problem* p, uint64_t* calls, double* out);
int orc_estimate_lipschitz_ex(const orc_factor* f, const orc_problem* p, double rel_tol, int max_rounds,
                              uint64_t* calls, double* out);
int orc_solve(const orc_problem* p, const orc_solver_config* cfg, int kind, const orc_factor* shared,
              orc_report** out);
int orc_solve_direct(const orc_problem* p, const orc_factor* f, const orc_solver_config* cfg,
                     int kind, const double* y0, const double* weight, orc_report** out);
int orc_warm_start(const orc_problem* p, const orc_factor* f, const orc_solver_config* cfg,
                   double lambda, double* y_out, uint64_t* dual_grad_calls);
void orc_report_free(orc_report* r);
int orc_report_summary_get(const orc_report* r, orc_report_summary* s);
int orc_report_arrays(const orc_report* r, double* x, double* u, double* y, double* z,
                      double* residual_trace, double* fbe_trace);
int orc_verify_report(const orc_problem* p, orc_report* r, const double* z_override);

/* CPU baseline timing (single thread, steady_clock): seconds per sweep */
int orc_time_sweeps(const orc_factor* f, const orc_problem* p, int nsweeps, int affine,
                    double* seconds);

#ifdef __cplusplus
}
#endif
#endif
