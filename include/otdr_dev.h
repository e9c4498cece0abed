/* otdr_dev.h -- C-ABI of the B200-native RDROT hot path (libotdr_dev.so).
 *
 * This is the drop-in boundary between the reference's C++ solver API
 * (/root/reference/proj/include/otdr/{problem,solver,regularizers,groups,duality}.hpp)
 * and the sm_100a kernels. Plain pointers and sizes only; every host buffer
 * is dense row-major fp64 like the reference's Eigen types (types.hpp:9) and
 * is copied in / out (value semantics, solver.hpp:74-87). An opaque context
 * owns all device memory, its CUDA stream, CUDA graphs and (for row-sharded
 * multi-GPU runs) its NCCL communicator.
 *
 * Entry point -> reference interface it replaces:
 *   otdr_dev_create / set_problem   Problem{cost,p,q}            problem.hpp:13-21
 *   otdr_dev_build_sqdist_cost      squared_distance_cost +      datagen.hpp:27, problem.hpp:29
 *                                   normalize_cost, on device
 *   otdr_dev_set_regularizer        ZeroReg / QuadraticReg /     regularizers.hpp:56-96,
 *                                   GroupLassoReg(column_class_blocks)   groups.hpp:34
 *   otdr_dev_set_state              make_state(problem, init)    solver.hpp:95-96
 *   otdr_dev_load_state             a SolverState value          solver.hpp:51-59
 *   otdr_dev_step                   step(state, problem, reg, rho) x iters   solver.hpp:99-100
 *   otdr_dev_solve                  solve(problem, reg, options) solver.hpp:102-103
 *   otdr_dev_get_state              SolverState fields           solver.hpp:51-59
 *   otdr_dev_objective              primal_objective             problem.hpp:32-33
 *   otdr_dev_duality_gap            duality_gap                  duality.hpp:31-32
 *   otdr_dev_get_trace              SolveReport::trace           solver.hpp:65-72
 *   otdr_dev_read_cost_otpb /       read_matrix_otpb /           io.cpp:127-158
 *   otdr_dev_write_plan_otpb        write_matrix_otpb (plan)
 *   otdr_dev_last_error             exception what() text        errors.hpp:9-34
 *
 * Errors: every call returns an otdr_status; the matching exception text of the
 * reference (e.g. "non-finite iterate at iteration 7 (check rho and
 * regularizer parameters)", solver.cpp:182-184) is available from
 * otdr_dev_last_error. There is no CPU fallback: without a CUDA device every
 * call that needs one returns OTDR_E_CUDA.
 *
 * Threading: a context is not thread-safe; distinct contexts may be driven from
 * distinct host threads.
 */
#ifndef OTDR_DEV_H
#define OTDR_DEV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OTDR_DEV_ABI_VERSION 1

typedef struct otdr_dev otdr_dev;

typedef enum {
  OTDR_OK = 0,
  OTDR_E_DIMENSION = 1,   /* DimensionMismatch       errors.hpp:10 */
  OTDR_E_NEGATIVE = 2,    /* NegativeEntry           errors.hpp:13 */
  OTDR_E_MARGINAL = 3,    /* MarginalSumOutOfRange   errors.hpp:16 */
  OTDR_E_ZERO_ITERS = 4,  /* ZeroIterations          errors.hpp:19 */
  OTDR_E_INVALID_ARG = 5, /* std::invalid_argument   solver.cpp:110-118 */
  OTDR_E_NONFINITE = 6,   /* NonFiniteIterate        errors.hpp:26 */
  OTDR_E_UNSUPPORTED = 7, /* regularizer/partition the kernels do not cover */
  OTDR_E_CUDA = 8,
  OTDR_E_NCCL = 9,
  OTDR_E_STATE = 10       /* call order (e.g. solve before set_problem) */
} otdr_status;

typedef enum { OTDR_REG_NONE = 0, OTDR_REG_QUAD = 1, OTDR_REG_GROUP_LASSO = 2 } otdr_reg_kind;

/* Device storage of C and X. Arithmetic is always fp64 in registers.
 * F64 reproduces the reference's element-wise rounding exactly;
 * F32 halves HBM traffic (12 B per plan entry per iteration). */
typedef enum { OTDR_STORE_F32 = 0, OTDR_STORE_F64 = 1 } otdr_storage;

typedef enum {
  OTDR_TERM_CONVERGED = 0, /* Termination::Converged solver.hpp:61 */
  OTDR_TERM_MAXITER = 1,
  OTDR_TERM_STALLED = 2
} otdr_termination;

typedef struct {
  int device;           /* CUDA ordinal */
  otdr_storage storage;
  int64_t m, n;         /* GLOBAL plan shape */
  /* Row sharding (nranks == 1: whole plan on this device). Rank r owns global
   * rows [row_begin, row_end); the n-vector of column sums and the three
   * residual scalars are ncclAllReduce'd once per iteration. */
  int rank, nranks;
  int64_t row_begin, row_end;
  const unsigned char* nccl_id; /* 128-byte ncclUniqueId, or NULL. nranks > 1 needs an NCCL id
                                  or a peer link (otdr_dev_peer_*) before the first exchange;
                                  for nranks == 1 it runs the NCCL exchange path on one GPU */
} otdr_dev_config;

typedef struct {
  double rho;           /* <= 0: default_stepsize 2/(m+n)      solver.cpp:55-57 */
  int64_t max_iter;     /* > 0 else OTDR_E_ZERO_ITERS          solver.cpp:106-109 */
  double tol_primal;    /* > 0                                 solver.cpp:113 */
  int has_tol_gap;
  double tol_gap;       /* > 0 when has_tol_gap                solver.cpp:116 */
  int64_t check_every;  /* > 0                                 solver.cpp:110 */
  int deterministic;    /* trace elapsed_ms = 0 (reductions are always fixed-order) */
  int record_trace;
  int fused;            /* even/odd sweep: odd iterations never read C  solver.cpp:127-177 */
} otdr_solve_opts;

typedef struct {
  int64_t iterations;   /* SolveReport::iterations = state.k */
  int termination;      /* otdr_termination */
  double rho;
  double r_primal;      /* max(||r||_2, ||s||_2) of the last iterate */
  double objective;     /* <C,X> + h(X)                        solver.cpp:239 */
  int64_t support_last_change; /* -1 unless record_trace */
  int64_t trace_rows;
  double device_ms;     /* device time of the iteration loop (CUDA events) */
} otdr_solve_result;

typedef struct {
  int64_t iter;
  double r_primal, gap, dual_residual;
  int64_t support;
  double elapsed_ms;
} otdr_trace_row;

typedef struct {
  double dual_value, gap, dual_residual;
} otdr_certificate;

/* Per-kernel device time of the last otdr_dev_profile call. */
typedef struct {
  double sweep_ms, reduce_ms, exchange_ms, update_ms; /* averages per iteration */
  int64_t iterations;
  double sweep_bytes;   /* algorithmic HBM bytes of one sweep (C, X read; X write) */
} otdr_kernel_times;

int otdr_dev_abi_version(void);
otdr_status otdr_dev_create(const otdr_dev_config* cfg, otdr_dev** out);
void otdr_dev_destroy(otdr_dev* ctx);
const char* otdr_dev_last_error(const otdr_dev* ctx);
/* 1 if a CUDA device is present (no context needed). */
int otdr_dev_cuda_available(void);

/* Local rows of C (row_end-row_begin) x n, p (local rows), q (n). The caller
 * validated them (validate_problem); values are stored at cfg->storage. */
otdr_status otdr_dev_set_problem(otdr_dev* ctx, const double* cost_rm, const double* p,
                                 const double* q);
/* C_ij = 0.5 ||a_i - b_j||^2 built on device in fp64 (datagen.cpp:43-54), then
 * divided by its global max (problem.cpp:68-74) unless all-zero. src_pts holds
 * the LOCAL rows' points (local_m x d), tgt_pts all n points (n x d). p, q as
 * in set_problem. *all_zero reports normalize_cost's flag (may be NULL). */
otdr_status otdr_dev_build_sqdist_cost(otdr_dev* ctx, const double* src_pts,
                                       const double* tgt_pts, int d, const double* p,
                                       const double* q, int* all_zero);
/* row_labels (local rows; -1 = row in no group) define GroupLassoReg over
 * column_class_blocks(row_labels, n): one group per (column, class). */
otdr_status otdr_dev_set_regularizer(otdr_dev* ctx, otdr_reg_kind kind, double param,
                                     const int32_t* row_labels);
/* make_state. X0/phi0/psi0 all NULL -> default_init. */
otdr_status otdr_dev_set_state(otdr_dev* ctx, const double* X0, const double* phi0,
                               const double* psi0);
/* Loads a complete SolverState (e.g. one a caller stepped elsewhere): X, phi,
 * a, r local rows; psi, b, s length n; theta, eta, k scalars. */
otdr_status otdr_dev_load_state(otdr_dev* ctx, const double* X, const double* phi,
                                const double* psi, const double* a, const double* b,
                                const double* r, const double* s, double theta, double eta,
                                int64_t k);
/* OTPB plan I/O straight from / to device buffers (io.cpp:127-158 format:
 * 16-byte header "OTPB", u32 m, u32 n, 4 zero bytes, then m*n fp64
 * row-major). read: the local rows of an m x n cost file become C (values
 * checked finite and >= 0 -> OTDR_E_NEGATIVE, shape -> OTDR_E_DIMENSION,
 * bad magic / truncation -> OTDR_E_INVALID_ARG); p, q as in set_problem.
 * write: the local rows of the current plan X land at their global offset,
 * so the ranks of a row-sharded run write one file together (the rank owning
 * row 0 writes the header). */
otdr_status otdr_dev_read_cost_otpb(otdr_dev* ctx, const char* path, const double* p,
                                    const double* q);
otdr_status otdr_dev_write_plan_otpb(otdr_dev* ctx, const char* path);
/* iters raw DR steps (no stopping logic), like calling step() iters times;
 * one persistent launch when the streaming / resident kernels apply. */
otdr_status otdr_dev_step(otdr_dev* ctx, double rho, int64_t iters);
/* Runs the solve loop from the current state with the reference's stopping
 * semantics, device-resident (one persistent kernel launch for the whole
 * loop, or a CUDA-graph while loop for traces; no per-iteration host round
 * trip), then evaluates the objective. */
otdr_status otdr_dev_solve(otdr_dev* ctx, const otdr_solve_opts* opts, otdr_solve_result* res);
/* Any pointer may be NULL. Local rows for X/phi/a/r; full length n for psi/b/s. */
otdr_status otdr_dev_get_state(otdr_dev* ctx, double* X, double* phi, double* psi, double* a,
                               double* b, double* r, double* s, double* theta, double* eta,
                               int64_t* k);
otdr_status otdr_dev_objective(otdr_dev* ctx, double* out);
otdr_status otdr_dev_duality_gap(otdr_dev* ctx, double rho, otdr_certificate* out);
otdr_status otdr_dev_get_trace(otdr_dev* ctx, otdr_trace_row* rows, int64_t cap, int64_t* count);
/* Times `iters` raw steps kernel by kernel with CUDA events on the context
 * stream (diagnostics for the roofline); state advances by iters. */
otdr_status otdr_dev_profile(otdr_dev* ctx, double rho, int64_t iters, otdr_kernel_times* out);
/* Device time (CUDA events on the context stream) of `iters` raw steps on the
 * configured device loop (one persistent launch, or graphs); state advances
 * by iters. */
otdr_status otdr_dev_time_steps(otdr_dev* ctx, double rho, int64_t iters, double* ms);
/* ---------------------------------------------------------------- peers
 * Peer-memory exchange of row-sharded runs: every rank exports a CUDA IPC
 * handle of its receive buffer, the handles are all-gathered by the caller
 * (any transport: torch.distributed, MPI, a file), and every rank imports all
 * of them. From then on the solve loop's per-iteration exchange runs inside
 * the streaming kernel over NVLink P2P stores (column sums as soon as each
 * stripe of the sweep is complete; epoch flags at system scope) instead of an
 * ncclAllReduce between kernels. Replaces the reference's single-process
 * loop (solver.cpp:104-241); there is no reference counterpart to bind. */
#define OTDR_PEER_HANDLE_BYTES 64
otdr_status otdr_dev_peer_export(otdr_dev* ctx, void* handle /* OTDR_PEER_HANDLE_BYTES */);
otdr_status otdr_dev_peer_import(otdr_dev* ctx, const void* handles /* nranks x 64, rank order */);
/* Same, for the ranks of one process (contexts ctxs[r] = rank r); used to
 * test the multi-rank path with several contexts on one GPU. */
otdr_status otdr_dev_peer_link_local(otdr_dev** ctxs, int nranks);

/* Number of kernel launches one DR iteration issues on the graph path
 * (sweep, reduce, update); 0 when iterations run inside one persistent
 * launch (on-chip resident or streaming solve kernel). */
int otdr_dev_kernels_per_iteration(const otdr_dev* ctx);
/* Which device loop step()/solve() use for the current configuration
 * (no certificate / trace / fused): OTDR_PATH_* below. */
enum { OTDR_PATH_GRAPH = 0, OTDR_PATH_RESIDENT = 1, OTDR_PATH_STREAM = 2 };
int otdr_dev_solve_path(const otdr_dev* ctx);
/* Human-readable name of the kernel step()/solve() launch in the current
 * configuration (e.g. "stream_kernel<f32, quad, sign-screened>"), for logs and
 * benchmark records; the string lives as long as the context. */
const char* otdr_dev_kernel_name(const otdr_dev* ctx);

/* ---------------------------------------------------------------- batched
 * B independent problems of one shape solved by ONE launch, each problem owned
 * by a thread-block cluster that keeps its C and X in (distributed) shared
 * memory for the whole solve. Equivalent to B sequential solve() calls from
 * default_init (solver.cpp:104-241) -- the GAN minibatch loop of the paper
 * (ot_cost_gradient, duality.cpp:26-31). Zero / quadratic
 * regularizers; shapes whose per-problem tiles exceed a 16-CTA cluster return
 * OTDR_E_UNSUPPORTED (callers then run per-problem contexts). */
typedef struct otdr_batch otdr_batch;
otdr_status otdr_batch_create(int device, otdr_storage storage, int64_t batch, int64_t m,
                              int64_t n, otdr_batch** out);
void otdr_batch_destroy(otdr_batch* bt);
const char* otdr_batch_last_error(const otdr_batch* bt);
/* costs B x m x n, p B x m, q B x n (each problem validated by the caller). */
otdr_status otdr_batch_set_problems(otdr_batch* bt, const double* costs, const double* p,
                                    const double* q);
/* per-problem squared-distance costs normalised by their own max
 * (gaussian_problem per seed): src B x m x d, tgt B x n x d. */
otdr_status otdr_batch_build_sqdist_costs(otdr_batch* bt, const double* src, const double* tgt,
                                          int d, const double* p, const double* q);
otdr_status otdr_batch_set_regularizer(otdr_batch* bt, otdr_reg_kind kind, double alpha);
/* results: B entries. opts->fused / record_trace / has_tol_gap unsupported. */
otdr_status otdr_batch_solve(otdr_batch* bt, const otdr_solve_opts* opts,
                             otdr_solve_result* results);
/* any pointer may be NULL: X B x m x n, phi B x m, psi B x n. */
otdr_status otdr_batch_get_plans(otdr_batch* bt, double* X, double* phi, double* psi);
/* The complete final SolverState of every problem (solver.hpp:51-59, owned by
 * each SolveReport, solver.hpp:74-87) -- what B sequential solve() calls
 * return. Any pointer may be NULL: X B x m x n; phi, a, r B x m; psi, b, s
 * B x n; theta, eta, k B entries. */
otdr_status otdr_batch_get_state(otdr_batch* bt, double* X, double* phi, double* psi, double* a,
                                 double* b, double* r, double* s, double* theta, double* eta,
                                 int64_t* k);

#ifdef __cplusplus
}
#endif
#endif /* OTDR_DEV_H */
