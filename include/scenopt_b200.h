/* SPDX-License-Identifier: MIT
 *
 * scenopt_b200 — C-ABI of the B200-native MINFBE / NAMA hot path.
 *
 * This is the drop-in boundary for the reference library's solver path
 * (arXiv 2107.01745 reference, /root/reference/proj/include/scenopt/). The
 * reference is a header-only C++ API with Eigen value types and exceptions;
 * it has no FFI layer of its own. Every entry point below replaces one
 * reference function (cited per declaration) with plain pointers and sizes:
 *   - 0 = success; a negative status maps 1:1 onto the reference exception
 *     types of errors.hpp:9-80 (the C++ shim include/scenopt_b200.hpp
 *     rethrows the same types), plus CUDA/NCCL/allocation failures;
 *   - scenopt_last_error() returns the message of the calling thread's last
 *     failure;
 *   - inputs are never retained; outputs are caller-owned buffers;
 *   - a scenopt_dev handle owns its device memory and one CUDA stream and is
 *     not thread-safe; distinct handles may be used concurrently.
 * There is no CPU fallback: device entry points fail with
 * SCENOPT_E_NODEVICE when no B200 (sm_100) device is present.
 *
 * Memory layouts follow the reference exactly (column-major, node-indexed):
 *   PrimalPoint.x  nx x num_nodes     (problem_data.hpp:64-67)
 *   PrimalPoint.u  nu x first_leaf
 *   dual vectors   stage blocks of nodes 1..n-1 in id order, then terminal
 *                  blocks of leaves in id order (problem_data.hpp:84-87,126-140)
 */
#ifndef SCENOPT_B200_H
#define SCENOPT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SCENOPT_ABI_VERSION 2

/* errors.hpp:9-80 */
enum scenopt_status {
  SCENOPT_OK = 0,
  SCENOPT_E_ERROR = -1,
  SCENOPT_E_NON_STOCHASTIC_MATRIX = -2,
  SCENOPT_E_STAGE_OUT_OF_RANGE = -3,
  SCENOPT_E_DIMENSION_MISMATCH = -4,
  SCENOPT_E_UNSUPPORTED_SPEC = -5,
  SCENOPT_E_NOT_STRONGLY_CONVEX = -6,
  SCENOPT_E_SHAPE_CHANGED = -7,
  SCENOPT_E_CACHE_MISMATCH = -8,
  SCENOPT_E_LINE_SEARCH_STALLED = -9,
  SCENOPT_E_STEP_UNDERFLOW = -10,
  SCENOPT_E_ZERO_PROBABILITY = -11,
  SCENOPT_E_INVALID_PARAMS = -12,
  SCENOPT_E_INFINITE_CONJUGATE = -13,
  SCENOPT_E_PARSE_ERROR = -14,
  SCENOPT_E_CUDA = -20,
  SCENOPT_E_NCCL = -21,
  SCENOPT_E_NOMEM = -22,
  SCENOPT_E_NODEVICE = -23
};

/* I/O flag for entry points that take vectors: buffers are host memory
 * (copied in/out inside the call) instead of device memory of the handle's
 * device. */
#define SCENOPT_HOST_IO 1

/* Flat, node-indexed problem description (ProblemInstance,
 * problem_data.hpp:95-141). Per-node arrays have one slot per node with slot
 * 0 (the root) unused; per-leaf arrays are indexed by leaf ordinal. All
 * matrices column-major. The tree must be BFS ordered (scenario_tree.hpp:
 * 228-238), which makes every node's children a contiguous id range. */
typedef struct scenopt_problem_view {
  int32_t nx, nu, num_stages, num_nodes;
  const int32_t* ancestor;      /* [n], -1 at the root */
  const double* probability;    /* [n] */
  const int32_t* stage_offsets; /* [num_stages + 2] */
  const double* root_state;     /* [nx] */
  const double *A, *B, *c;      /* [n][nx*nx], [n][nx*nu], [n][nx] (NodeDynamics) */
  const double *Q, *R, *S;      /* [n][nx*nx], [n][nu*nu], [n][nu*nx] (NodeCost) */
  const double *q, *r;          /* [n][nx], [n][nu] */
  const int32_t* stage_rows;    /* [n], rows of F_i/G_i (0 at the root) */
  const double *F, *G;          /* node i's block at dual_offset[i]*nx / dual_offset[i]*nu */
  const int32_t* g_kind;        /* [n] NonsmoothKind: 0 None, 1 Box, 2 ScaledL1 */
  const double* g_gamma;        /* [n] */
  const double *P, *p;          /* [L][nx*nx], [L][nx] (TerminalCost) */
  const int32_t* terminal_rows; /* [L] */
  const double* FN;             /* leaf l's block at (tdual_offset[l] - stage_rows_total)*nx */
  const int32_t* tg_kind;       /* [L] */
  const double* tg_gamma;       /* [L] */
  const double *zmin, *zmax;    /* [dual_dim] box bounds in dual layout */
} scenopt_problem_view;

/* SolverConfig, solvers.hpp:28-46. backtracking_rule: 0 Original,
 * 1 Simple, 2 None. */
typedef struct scenopt_solver_config {
  double lambda0, eps, eps_curv, eps_bt, beta_bt;
  int32_t memory, max_iters, backtracking_rule, warm_start, warm_start_iters, precondition,
      nama_parallel_linesearch, nama_update_tlambda;
} scenopt_solver_config;

/* Scalar part of SolverReport, solvers.hpp:66-84 (+ OracleStats,
 * tree_oracles.hpp:14-21). status: 0 Converged, 1 MaxItersExceeded. */
typedef struct scenopt_report_summary {
  int32_t status, iterations, verified, trace_len;
  uint64_t dual_grad_calls, hessian_vec_calls, prox_calls, conj_calls, lipschitz_calls;
  double lipschitz_estimate, lambda_final, eps, residual_inf, wall_ms, verify_residual_inf,
      verify_subdiff_dist;
} scenopt_report_summary;

/* Device handle facts used by the benchmark's roofline accounting. */
typedef struct scenopt_dev_info {
  int32_t device, sm_count, grid_ctas, ctas_per_sm, slots, items_bw, items_fw, nodes_per_item_max;
  int64_t slot_bytes, matrix_bytes_bw, matrix_bytes_fw, device_bytes;
  int64_t sweep_bytes_hom, sweep_bytes_aff, sweep_bytes_hom2; /* algorithmic bytes per sweep */
  int32_t cut_stage;   /* CTA subtree-ownership cut of the main region; -1: all global tickets */
  int32_t shard_stage; /* subtree sharding over ranks: cut stage, -1 when not sharded */
  int32_t rank, world; /* this handle's rank in the shard group (0, 1 when not sharded) */
  int32_t shard_first, shard_past; /* this rank's shard-stage node ids [first, past) */
  int32_t items_global;   /* items too large for a shared-memory slot (blocks read from HBM in place) */
  int32_t consumer_stage; /* 1: vectors staged by the consumer teams (very wide states) */
  int32_t flat_top;       /* 1: forward stages above the cut flattened into one level */
  int32_t device_factor;  /* 1: factor computed on the device (scenopt_dev_create_device_factor) */
  int32_t producer_warps; /* sweep kernel geometry: 4, or 6 for layouts of many-node items */
  int64_t exchange_doubles; /* sharded: doubles sum-allreduced per sweep and right-hand side; 0 otherwise */
} scenopt_dev_info;

typedef struct scenopt_problem scenopt_problem;
typedef struct scenopt_factor scenopt_factor;
typedef struct scenopt_dev scenopt_dev;
typedef struct scenopt_report scenopt_report;
typedef struct scenopt_lbfgs scenopt_lbfgs;

const char* scenopt_last_error(void);
int scenopt_abi_version(void);
int scenopt_device_count(void); /* sm_100 devices visible; 0 on a GPU-less host */

/* ---- problem (host) ---------------------------------------------------- */
/* ProblemInstance + finalize_layout(), problem_data.hpp:95-141 */
int scenopt_problem_create(const scenopt_problem_view* v, scenopt_problem** out);
/* gen_random_instance, generators.hpp:255-328, with per-stage branching
 * br[t] (1 after the listed stages); nbranch == 1 and horizon entries equal
 * reproduce the reference's full-branching tree. */
int scenopt_problem_gen_random(uint64_t seed, int nx, int nu, int horizon, const int32_t* branching,
                               int nbranch, scenopt_problem** out);
/* One shard's part of the same instance (B200 extension for subtree-sharded
 * runs): the random stream is drawn in full in the reference's order, but
 * only the nodes rank `rank` of `world` holds (its subtrees under the plan
 * of scenopt_shard_plan, the stages above and the shard-stage nodes) are
 * built; their values equal the full instance's bit for bit. Every dual row
 * is complete. The result can only build that rank's sharded handle with a
 * device factor (scenopt_dev_create_sharded[_group] with f == NULL). */
int scenopt_problem_gen_random_shard(uint64_t seed, int nx, int nu, int horizon, const int32_t* branching,
                                     int nbranch, int world, int rank, int shard_stage, scenopt_problem** out);
/* SpringMassParams, generators.hpp:49-64. Arrays of length 0 take the
 * reference defaults (generators.hpp:149-162); transition is row-major. */
typedef struct scenopt_spring_mass_params {
  double mass_kg, stiffness, damping, input_bound, velocity_bound;
  int32_t horizon;
  double sampling, state_weight, input_weight, terminal_weight;
  int32_t initial_len, transition_rows, transition_cols, mode_values_len, root_state_len;
  const double* initial_probs;
  const double* transition;
  const double* mode_values;
  const double* root_state;
} scenopt_spring_mass_params;
/* the member defaults of SpringMassParams (generators.hpp:50-59), empty arrays */
void scenopt_spring_mass_defaults(scenopt_spring_mass_params* par);
/* gen_spring_mass, generators.hpp:119-218: ZOH-discretized spring-mass-damper
 * array (nx = 2M, nu = M-1) on the Markov mode tree (build_from_markov,
 * scenario_tree.hpp:72-126). par == NULL: defaults. */
int scenopt_problem_gen_spring_mass(int masses, const scenopt_spring_mass_params* par, scenopt_problem** out);
/* detail::spring_mass_continuous, generators.hpp:70-91: A (2M x 2M), B (2M x M-1), column-major */
int scenopt_spring_mass_continuous(int masses, const scenopt_spring_mass_params* par, double* A, double* B);
/* discretize_zoh, generators.hpp:97-112 (exp of [[A, B], [0, 0]]·period), column-major */
int scenopt_discretize_zoh(const double* A, const double* B, int n, int m, double period, double* Ad, double* Bd);
/* matrix exponential (Eigen MatrixBase::exp semantics: Pade scaling and squaring), column-major n x n */
int scenopt_expm(const double* X, int n, double* out);
/* sample_initial_state, generators.hpp:223-234: `count` consecutive draws from
 * std::mt19937_64(seed), each 2M doubles, into out */
int scenopt_sample_initial_states(int masses, const scenopt_spring_mass_params* par, uint64_t seed, int count,
                                  double* out);
/* ---- problem files, problem_io.hpp:18-559 ("scenopt-problem-v1" JSON) ---- */
/* serialize_problem (:480): canonical text (sorted keys, 2-space indent, "\n"
 * terminated). buf == NULL queries the length (*len, without the NUL); then
 * call again with cap >= *len + 1. */
int scenopt_problem_serialize(scenopt_problem* p, char* buf, size_t cap, size_t* len);
/* parse_problem (:484) / problem_from_json (:323): SCENOPT_E_PARSE_ERROR on
 * malformed JSON, a wrong schema, missing keys, ragged data, or an instance
 * that fails validation (message lists every violation). */
int scenopt_problem_parse(const char* text, size_t len, scenopt_problem** out);
/* validate_problem_text (:512): number of violations (0: parses and
 * validates), messages joined by '\n' into buf */
int scenopt_problem_validate_text(const char* text, size_t len, char* buf, int buflen);
int scenopt_problem_save(const scenopt_problem* p, const char* path);  /* save_problem (:494) */
int scenopt_problem_load(const char* path, scenopt_problem** out);    /* load_problem (:502) */
/* content_hash (:539) and factor_hash (:546): FNV-1a of the canonical text /
 * of the factor-determining fields (no root state, modes or nonsmooth specs) */
int scenopt_problem_hashes(const scenopt_problem* p, uint64_t* content, uint64_t* factor);
/* ScenarioTree::mode (scenario_tree.hpp:41): per-node Markov mode, -1 at the
 * root; empty when unknown. get returns the count (0: none). */
int scenopt_problem_set_mode(scenopt_problem* p, const int32_t* mode, int n);
int scenopt_problem_get_mode(const scenopt_problem* p, int32_t* out, int cap);
/* Pointers into the handle's own arrays (valid until destroy). */
int scenopt_problem_get_view(scenopt_problem* p, scenopt_problem_view* v, int32_t* dual_dim);
/* dims = {nx, nu, num_stages, num_nodes, num_leaves, first_leaf, dual_dim, primal_dim} */
int scenopt_problem_dims(const scenopt_problem* p, int32_t* dims);
/* validate(ProblemInstance), problem_data.hpp:233-314: returns the number of
 * violations, messages joined by '\n' into buf. */
int scenopt_problem_validate(const scenopt_problem* p, char* buf, int buflen);
/* precondition(), solvers.hpp:569-602 */
int scenopt_problem_precondition(const scenopt_problem* p, scenopt_problem** out);
void scenopt_problem_destroy(scenopt_problem* p);

/* ---- factor (host, offline) -------------------------------------------- */
/* factor(), riccati.hpp:82-182 */
int scenopt_factor_create(const scenopt_problem* p, scenopt_factor** out);
/* refactor_affine(), riccati.hpp:187-216 */
int scenopt_refactor_affine(scenopt_factor* f, const scenopt_problem* p);
/* FactorCache members, flattened (same layout as the oracle export). */
int scenopt_factor_export(const scenopt_factor* f, double* gain, double* child_to_input,
                          double* closed_loop, double* dual_to_input, double* dual_to_costate,
                          double* input_affine, double* costate_affine, double* value_quad,
                          double* leaf_costate_affine);
void scenopt_factor_destroy(scenopt_factor* f);

/* ---- device handle ----------------------------------------------------- */
/* factor() on the device (riccati.hpp:82-182): the
 * handle is packed from problem data only and the Riccati factor is computed
 * by a per-stage GPU kernel directly into the sweep layout (no host factor,
 * no factor upload). Throws NotStronglyConvex like factor(). */
int scenopt_dev_create_device_factor(const scenopt_problem* p, int device, scenopt_dev** out);
/* Recompute the device factor of the handle's problem data in place (the
 * factor kernels only; e.g. after the handle's data were updated). */
int scenopt_dev_refactor_device(scenopt_dev* d);
/* refactor_affine (riccati.hpp:187-216) on the device, for MPC-style
 * re-solves: only p's linear terms (q, r, c, p_N) and root state move to the
 * device (O(n (nx+nu)) bytes) and the affine factor terms are recomputed in
 * place; the matrices of p must be those the handle was factored with.
 * Requires a handle from scenopt_dev_create_device_factor. */
int scenopt_dev_refactor_affine(scenopt_dev* d, const scenopt_problem* p);
/* The device factor in scenopt_factor_export's layout (p: the handle's problem). */
int scenopt_dev_factor_export(scenopt_dev* d, const scenopt_problem* p, double* gain, double* child_to_input,
                              double* closed_loop, double* dual_to_input, double* dual_to_costate,
                              double* input_affine, double* costate_affine, double* value_quad,
                              double* leaf_costate_affine);
/* Packs (ProblemInstance, FactorCache) into the stage-major device layout and
 * uploads it. */
int scenopt_dev_create(const scenopt_problem* p, const scenopt_factor* f, int device,
                       scenopt_dev** out);
/* Subtree-sharded handle: rank `rank` of `world` processes
 * (one per GPU, all calling this concurrently) owns the subtrees of a
 * contiguous, byte-balanced range of the shard-stage nodes (shard_stage < 0:
 * the smallest stage with >= world nodes) and replicates the stages above.
 * Primal and dual vectors are sharded the same way: a rank holds valid
 * values on its own nodes / rows and on the replicated top. Every sweep
 * sum-allreduces one exchange buffer (the shard-stage nodes' contributions
 * to their parents and their dual rows); every reduction of the dual-space
 * kernels allgathers the ranks' partial sums (a few dozen doubles) and
 * combines them in rank order on the device, so every rank takes identical
 * decisions. Device outputs of scenopt_dev_sweep[_async] are rank-local;
 * host outputs of the public entry points and solver reports are assembled
 * in full. nccl_id: 128 bytes from scenopt_nccl_unique_id() on one rank,
 * shared with the others (NULL: no communicator, see the phase API below;
 * world == 1 needs none). The same problem and factor must be passed on
 * every rank. Replaces nothing in the reference (single-process); every
 * other entry point accepts the sharded handle (solvers: memory <= 6;
 * scenopt_linesearch_cert with explicit trials: unsharded handles only).
 * f == NULL: the factor is computed on the device (K9): each rank factors
 * its own subtrees, the shard-stage value matrices are exchanged in one
 * sum-allreduce, and every rank factors the replicated top; no rank needs a
 * host factor. */
int scenopt_nccl_unique_id(void* out128);
/* Host-only plan of the above: the shard stage actually used and the
 * world + 1 bounds of the ranks' shard-stage node ranges. */
int scenopt_shard_plan(const scenopt_problem* p, int world, int shard_stage, int32_t* stage_out,
                       int32_t* bounds);
/* Host-only: the dual rows rank `rank` counts in the sharded reductions
 * (counted[i] = 1: a stage or terminal row of its subtrees, or a top row on
 * rank 0), dual_dim bytes. */
int scenopt_shard_rows(const scenopt_problem* p, int world, int shard_stage, int rank, uint8_t* counted);
int scenopt_dev_create_sharded(const scenopt_problem* p, const scenopt_factor* f, int device, int rank,
                               int world, int shard_stage, const void* nccl_id, scenopt_dev** out);
/* Emulated shard group: `world` sharded handles of ONE process, driven by one
 * host thread per rank, exchange through host memory after a stream
 * synchronisation (no NCCL; kernels of different ranks never wait on one
 * another, so several ranks can share one GPU). For tests of the sharded
 * solver on one device. */
typedef struct scenopt_shard_group scenopt_shard_group;
int scenopt_shard_group_create(int world, scenopt_shard_group** out);
void scenopt_shard_group_destroy(scenopt_shard_group* g);
int scenopt_dev_create_sharded_group(const scenopt_problem* p, const scenopt_factor* f, int device, int rank,
                                     scenopt_shard_group* g, int shard_stage, scenopt_dev** out);
/* Sharded handles created with nccl_id == NULL leave the exchange to the
 * caller (emulating ranks on one device, tests): phase 0 zeroes the Hx rows
 * this rank does not write, runs the local backward and writes this rank's
 * shard-stage contributions and dual rows into the exchange buffer (zeros
 * elsewhere); the caller sums the buffers over ranks into every rank's
 * buffer; phase 1 runs the top backward and all forward work and zeroes the
 * replicated top rows of Hx on ranks != 0, so the sum of the ranks' Hx is
 * the full Hx. Device pointers, handle stream. */
int scenopt_shard_sweep_phase(scenopt_dev* d, int phase, int nrhs, int affine, const double* const* y,
                              double* const* Hx);
int scenopt_shard_exchange_buffer(scenopt_dev* d, double** buf, size_t* doubles_per_rhs);
int scenopt_dev_info_get(const scenopt_dev* d, scenopt_dev_info* info);
int scenopt_dev_synchronize(scenopt_dev* d);
/* The handle's CUDA stream (cudaStream_t) for event timing by callers. */
int scenopt_dev_stream(scenopt_dev* d, void** stream);
void scenopt_dev_destroy(scenopt_dev* d);
/* Device scratch the caller may use for device-resident I/O (bench). */
int scenopt_dev_alloc(scenopt_dev* d, size_t bytes, void** out);
int scenopt_dev_free(scenopt_dev* d, void* ptr);
int scenopt_dev_memcpy(scenopt_dev* d, void* dst, const void* src, size_t bytes, int kind);

/* ---- oracles: tree_oracles.hpp:33-129 ----------------------------------- */
/* One fused backward/forward sweep with apply_H in the epilogue for nrhs
 * (1 or 2) right-hand sides. affine = 1: dual_grad (x(y)); 0: hessian_vec
 * (x0(r)). x/u/Hx entries may be NULL to skip that output. */
int scenopt_dev_sweep(scenopt_dev* d, int nrhs, int affine, const double* const* y,
                      double* const* x, double* const* u, double* const* Hx, int flags);
/* Same, enqueued on the handle's stream without a host synchronisation
 * (device pointers only). */
int scenopt_dev_sweep_async(scenopt_dev* d, int nrhs, int affine, const double* const* y,
                            double* const* x, double* const* u, double* const* Hx);
/* dual_grad / hessian_vec, tree_oracles.hpp:96-114 */
int scenopt_dual_grad(scenopt_dev* d, const double* y, double* x, double* u, int flags);
int scenopt_hessian_vec(scenopt_dev* d, const double* r, double* x, double* u, int flags);
/* apply_H, problem_data.hpp:144-162 */
int scenopt_apply_H(scenopt_dev* d, const double* x, const double* u, double* z, int flags);
/* fhat_value, tree_oracles.hpp:125-129 */
int scenopt_fhat_value(scenopt_dev* d, const double* y, double* out, int flags);

/* ---- nonsmooth term: prox.hpp:58-171 ------------------------------------ */
int scenopt_prox_g(scenopt_dev* d, const double* v, double gamma_prox, double* out, int flags);
int scenopt_conj_value_g(scenopt_dev* d, const double* w, double* out, int flags);
int scenopt_dist_subdiff_inf(scenopt_dev* d, const double* y, const double* z, double* out,
                             int flags);

/* ---- forward-backward machinery: fbe.hpp:22-231 ------------------------- */
/* fb_step: scalars = {fhat, conj_T, znorm_sq, value} */
int scenopt_fb_step(scenopt_dev* d, const double* y, double lambda, double* x, double* u,
                    double* Hx, double* z, double* R, double* T, double* scalars, int flags);
/* fbe_grad: grad = R + lambda H x0(R) */
int scenopt_fbe_grad(scenopt_dev* d, const double* R, double lambda, double* grad, int flags);
/* linesearch_cert (shift == NULL) / linesearch_cert_shifted + evaluate_cert
 * at ntau taus; identical contract to the oracle's orc_linesearch_cert. */
int scenopt_linesearch_cert(scenopt_dev* d, const double* y, const double* Hx, double lambda,
                            const double* state_scalars, const double* shift, const double* dir,
                            int ntau, const double* taus, double* deltas, double* cert_scalars,
                            double* cert_fhat, double* w, double* Hx_w, double* z, double* R,
                            double* T, int flags);

/* ---- L-BFGS: lbfgs.hpp:22-84 (device-resident pairs) -------------------- */
/* The buffer lives on d's device (d == NULL: a standalone buffer on device
 * 0, as LbfgsBuffer(memory, eps_curv) carries no problem); vectors are host
 * arrays of length n (fixed by the first call). */
int scenopt_lbfgs_create(scenopt_dev* d, int memory, double eps_curv, scenopt_lbfgs** out);
int scenopt_lbfgs_push(scenopt_lbfgs* b, int n, const double* step, const double* change,
                       double scale_ref); /* 1 accepted, 0 rejected, <0 error */
int scenopt_lbfgs_apply(scenopt_lbfgs* b, int n, const double* grad, double* out);
int scenopt_lbfgs_clear(scenopt_lbfgs* b);
int scenopt_lbfgs_size(const scenopt_lbfgs* b);
double scenopt_lbfgs_gamma0(const scenopt_lbfgs* b);
void scenopt_lbfgs_destroy(scenopt_lbfgs* b);

/* ---- solvers: solvers.hpp:89-720 ---------------------------------------- */
/* estimate_dual_lipschitz, solvers.hpp:89-113 */
int scenopt_estimate_lipschitz(scenopt_dev* d, uint64_t* calls, double* out);
/* The same with the reference's optional arguments (solvers.hpp:88-93):
 * stop when the Rayleigh quotient moves by <= rel_tol relative, or after
 * max_rounds sweeps (max_rounds <= 0: no sweep, 1e-12). */
int scenopt_estimate_lipschitz_ex(scenopt_dev* d, double rel_tol, int max_rounds, uint64_t* calls, double* out);
/* solve_minfbe (kind 0) / solve_nama (1) / solve_gpad (2) from y0 (host,
 * NULL = zeros), optional residual weight (host, NULL = none). */
int scenopt_dev_solve(scenopt_dev* d, const scenopt_solver_config* cfg, int kind, const double* y0,
                      const double* residual_weight, scenopt_report** out);
/* warm_start, solvers.hpp:545-564 */
int scenopt_warm_start(scenopt_dev* d, const scenopt_solver_config* cfg, double lambda,
                       double* y_out, uint64_t* dual_grad_calls);
/* solve(), solvers.hpp:645-720: precondition, factor (unless shared),
 * Lipschitz estimate, warm start, solver run, verify_report. */
int scenopt_solve(const scenopt_problem* p, const scenopt_solver_config* cfg, int kind,
                  const scenopt_factor* shared, int device, scenopt_report** out);
int scenopt_report_summary_get(const scenopt_report* r, scenopt_report_summary* s);
/* x [nx*n], u [nu*first_leaf], y/z [dual_dim], traces [trace_len]; NULL skips */
int scenopt_report_arrays(const scenopt_report* r, double* x, double* u, double* y, double* z,
                          double* residual_trace, double* fbe_trace);
/* verify_report, solvers.hpp:630-639, against problem p (z_override: host
 * dual vector replacing the report's z first, or NULL). */
int scenopt_verify_report(const scenopt_problem* p, scenopt_report* r, const double* z_override,
                          int device);
void scenopt_report_destroy(scenopt_report* r);

/* ---- experiment harness, experiment.hpp:22-283 -------------------------- */
typedef struct scenopt_experiment scenopt_experiment; /* RunReport */
/* ExperimentRow (:63-80); strings and the trace point into the report */
typedef struct scenopt_experiment_row {
  const char* instance_id;
  const char* solver;
  const char* error; /* "" unless the factorization or the solve threw */
  int32_t iterations;
  uint64_t dual_grad_calls, hessian_vec_calls, prox_calls;
  double final_residual_inf, wall_ms;
  int32_t converged, fbe_monotone, trace_len;
  const double* residual_trace;
} scenopt_experiment_row;
/* SolverSummary (:86-96) */
typedef struct scenopt_solver_summary {
  char solver[16];
  int32_t count, converged, fbe_violations;
  double median_calls, p84_calls, p95_calls, frac_within_50, total_wall_ms;
} scenopt_solver_summary;
/* run_experiment (:222-283): every solver ("minfbe", "nama", "pnama" = NAMA
 * with the parallel line search, "gpad") on every instance, in order, through
 * scenopt_solve on `device`. reuse_factors shares one factor per factor hash
 * (not with preconditioning). A run that fails with a scenopt error is
 * recorded in its row; CUDA / NCCL / allocation failures abort the batch. */
int scenopt_run_experiment(const scenopt_problem* const* problems, const char* const* ids, int count,
                           const char* const* solvers, int nsolvers, const scenopt_solver_config* cfg,
                           int include_timing, int reuse_factors, int device, scenopt_experiment** out);
int scenopt_experiment_row_count(const scenopt_experiment* x);
int scenopt_experiment_row_get(const scenopt_experiment* x, int i, scenopt_experiment_row* row);
/* which: 0 csv() (:137), 1 traces_csv() (:153), 2 summary_json().dump(2) + "\n"
 * (:194; metadata_json: a JSON object text or NULL). buf == NULL queries the length. */
int scenopt_experiment_text(scenopt_experiment* x, int which, const char* metadata_json, char* buf, size_t cap,
                            size_t* len);
/* summaries() (:163): returns the number of solvers, fills up to cap */
int scenopt_experiment_summaries(const scenopt_experiment* x, scenopt_solver_summary* out, int cap);
void scenopt_experiment_destroy(scenopt_experiment* x);
/* treebench's solve report (treebench.cpp:52-85): "scenopt-solvereport-v1"
 * JSON of one solve of problem p, dump(2) + "\n"; buf == NULL queries the length */
int scenopt_report_json(const scenopt_report* r, const scenopt_problem* p, const char* solver, int converged,
                        char* buf, size_t cap, size_t* len);

#ifdef __cplusplus
}
#endif
#endif /* SCENOPT_B200_H */
