/* otdr_oracle.h -- CPU restatement of the reference RDROT hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This library is the parity checker for the
 * B200 kernels in paper_2305_18483_b200/csrc. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it. The product
 * path (libotdr_dev.so) never links or calls it.
 *
 * It restates, in plain C++ without Eigen (Eigen is absent in this image, so the
 * reference itself cannot be compiled -- see DESIGN.md "Oracle"), the following
 * reference files (paths relative to /root/reference/proj):
 *   include/otdr/rng.hpp:14-45        mt19937_64 + 53-bit uniform + Box-Muller
 *   src/datagen.cpp:21-129            gaussian_problem / adaptation_problem
 *   src/problem.cpp:13-85             validate_problem / normalize_cost / objective
 *   src/regularizers.cpp:28-99        zero / quadratic / group-lasso
 *   src/groups.cpp:8-60               make_partition / column_class_blocks
 *   src/solver.cpp:15-256             make_state / step / solve / skip count
 *   src/duality.cpp:5-31              recover_duals / duality_gap
 *   tests/support/oracles.cpp:366-380 textbook DR (closed-form affine projection)
 *   tests/support/oracles.cpp:16-345  affine / polytope projection, projgrad_solve,
 *                                     LP vertex enumeration, transportation simplex
 *                                     (otdr_lp_oracles.cpp)
 *
 * All arrays are dense row-major fp64, caller-owned. Status codes equal the
 * product's otdr_status values (include/otdr_dev.h).
 */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORA_OK = 0,
  ORA_E_DIMENSION = 1,   /* DimensionMismatch        errors.hpp:10 */
  ORA_E_NEGATIVE = 2,    /* NegativeEntry            errors.hpp:13 */
  ORA_E_MARGINAL = 3,    /* MarginalSumOutOfRange    errors.hpp:16 */
  ORA_E_ZERO_ITERS = 4,  /* ZeroIterations           errors.hpp:19 */
  ORA_E_INVALID_ARG = 5, /* std::invalid_argument                   */
  ORA_E_NONFINITE = 6,   /* NonFiniteIterate         errors.hpp:26 */
  ORA_E_UNSUPPORTED = 7
};

enum { ORA_REG_NONE = 0, ORA_REG_QUAD = 1, ORA_REG_GROUP_LASSO = 2 };
enum { ORA_TERM_CONVERGED = 0, ORA_TERM_MAXITER = 1, ORA_TERM_STALLED = 2 };

typedef struct {
  int64_t m, n;
  const double* C; /* m*n */
  const double* p; /* m */
  const double* q; /* n */
} ora_problem;

/* Group lasso groups are CSR over (row, col) cells: cells[2*t], cells[2*t+1],
 * group g = cells [offsets[g], offsets[g+1]). groups.hpp:15-27. */
typedef struct {
  int kind;
  double param; /* alpha (quad) or lambda (group lasso) */
  int64_t num_groups;
  const int64_t* offsets; /* num_groups + 1 */
  const int32_t* cells;   /* 2 * offsets[num_groups] */
} ora_reg;

typedef struct {
  int64_t m, n;
  double* X;   /* m*n */
  double* phi; /* m */
  double* psi; /* n */
  double* a;   /* m */
  double* b;   /* n */
  double* r;   /* m */
  double* s;   /* n */
  double theta, eta;
  int64_t k;
} ora_state;

typedef struct {
  double rho; /* <= 0: default 2/(m+n) */
  int64_t max_iter;
  double tol_primal;
  int has_tol_gap;
  double tol_gap;
  int64_t check_every;
  int deterministic;
  int record_trace;
  int fused;
  int threads; /* OpenMP threads for the sweep (baseline timing); 1 = reference */
} ora_options;

typedef struct {
  int64_t iter;
  double r_primal, gap, dual_residual;
  int64_t support;
  double elapsed_ms;
} ora_trace_row;

typedef struct {
  double objective;
  int64_t iterations;
  int termination;
  double rho;
  double r_primal;
  int64_t support_last_change;
  int64_t trace_len;
} ora_report;

/* ---- rng.hpp ---- */
void* ora_rng_new(uint64_t seed);
void ora_rng_free(void* h);
double ora_rng_uniform01(void* h);
double ora_rng_normal(void* h);
uint64_t ora_rng_raw(void* h);

/* ---- datagen.cpp ---- */
void ora_gaussian_problem(int64_t m, int64_t n, uint64_t seed, double* C, double* p,
                          double* q, double* src_pts, double* tgt_pts);
int ora_adaptation_problem(int64_t m, int64_t n, int classes, uint64_t seed,
                           int identity_map, double* C, double* p, double* q,
                           double* src_pts, double* tgt_pts, int32_t* src_labels,
                           int32_t* tgt_labels);
void ora_squared_distance_cost(int64_t m, int64_t n, int64_t d, const double* a,
                               const double* b, double* C);

/* ---- problem.cpp ---- (validate renormalizes p, q in place) */
int ora_validate_problem(int64_t m, int64_t n, const double* C, double* p, double* q,
                         char* msg, int msglen);
int ora_normalize_cost(int64_t m, int64_t n, double* C, int* all_zero);
double ora_primal_objective(const ora_problem* pr, const double* X, const ora_reg* reg);

/* ---- groups.cpp ---- cells_out needs 2*m*n int32, offsets_out m*n+1 */
int ora_column_class_blocks(const int32_t* labels, int64_t m, int64_t n,
                            int32_t* cells_out, int64_t* offsets_out,
                            int64_t* num_groups_out);

/* ---- regularizers.cpp ---- */
void ora_prox(const ora_reg* reg, int64_t m, int64_t n, double* V, double rho);
double ora_reg_value(const ora_reg* reg, int64_t m, int64_t n, const double* X);

/* ---- solver.cpp ---- */
double ora_default_stepsize(int64_t m, int64_t n);
void ora_default_init(int64_t m, int64_t n, double* phi0, double* psi0);
/* X0/phi0/psi0 may all be NULL (default init). */
int ora_make_state(const ora_problem* pr, const double* X0, const double* phi0,
                   const double* psi0, ora_state* st, char* msg, int msglen);
void ora_step(ora_state* st, const ora_problem* pr, const ora_reg* reg, double rho,
              int threads);
/* st must come from ora_make_state (the warm start). */
int ora_solve(const ora_problem* pr, const ora_reg* reg, const ora_options* opt,
              ora_state* st, ora_report* rep, ora_trace_row* trace, int64_t trace_cap,
              char* msg, int msglen);
int64_t ora_compute_skip_count(const ora_problem* pr);

/* ---- duality.cpp ---- */
void ora_duality_gap(const ora_problem* pr, const ora_reg* reg, const ora_state* st,
                     double rho, double* dual_value, double* gap, double* dual_residual);

/* ---- tests/support/oracles.cpp:366-380 (closed-form projection) ---- */
/* xs, ys: iters*m*n each. y0: m*n. */
void ora_dr_reference(const ora_problem* pr, const ora_reg* reg, double rho,
                      const double* y0, int iters, double* xs, double* ys);

/* Algorithm-independent optimality oracles (otdr_lp_oracles.cpp;
 * tests/support/oracles.cpp:16-345). Dense row-major fp64. */
void ora_affine_project(int64_t m, int64_t n, const double* Z, const double* p, const double* q,
                        double* out);
void ora_polytope_project(int64_t m, int64_t n, const double* Z, const double* p, const double* q,
                          int max_iter, double tol, double* out);
int ora_lp_vertex_solve(int64_t m, int64_t n, const double* C, const double* p, const double* q,
                        double* X, double* value);
int ora_transport_simplex(int64_t m, int64_t n, const double* C, const double* p,
                          const double* q, double* X, double* value);
int ora_projgrad_solve(int64_t m, int64_t n, const double* C, const double* p, const double* q,
                       double alpha, double* X, double* gm);

#ifdef __cplusplus
}
#endif
