// otdr_oracle.cpp -- CPU restatement of the reference RDROT hot path.
//
// TEST INFRASTRUCTURE ONLY (the parity checker; see otdr_oracle.h). Nothing in
// the product library links this file.
//
// Every function cites the reference file:line it restates (paths relative to
// /root/reference/proj). Arithmetic order follows the reference expression
// trees term by term; compile with -ffp-contract=off so no FMA contraction
// changes the rounding (the reference builds for baseline x86-64, which has no
// FMA). Reductions run sequentially (Eigen's packet-wise redux order is not
// reproducible without Eigen; the reference's own tests pin the recurrence at
// 1e-9/1e-10, never bitwise).
#include "otdr_oracle.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <random>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr int64_t kStallWindow = 10000;       // solver.cpp:17
constexpr double kStallRelImprove = 1e-14;    // solver.cpp:18
constexpr double kMarginalRejectTol = 1e-6;   // problem.cpp:15
constexpr double kMarginalSkipTol = 1e-13;    // problem.cpp:18

void set_msg(char* msg, int len, const std::string& s) {
  if (msg && len > 0) {
    std::snprintf(msg, static_cast<size_t>(len), "%s", s.c_str());
  }
}

// ---------------------------------------------------------------- rng.hpp:14-45
struct Rng {
  std::mt19937_64 eng;
  bool have_spare = false;
  double spare = 0.0;
  explicit Rng(uint64_t seed) : eng(seed) {}
  double uniform01() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; }
  double normal() {
    if (have_spare) {
      have_spare = false;
      return spare;
    }
    const double u1 = static_cast<double>((eng() >> 11) + 1) * 0x1.0p-53;
    const double u2 = uniform01();
    const double rad = std::sqrt(-2.0 * std::log(u1));
    const double ang = 2.0 * kPi * u2;
    spare = rad * std::sin(ang);
    have_spare = true;
    return rad * std::cos(ang);
  }
};

// ------------------------------------------------------ regularizers.cpp:49-99
// Applies prox_{rho h} in place to the m x n row-major matrix V.
void prox_in_place(const ora_reg* reg, int64_t m, int64_t n, double* V, double rho,
                   int threads) {
  (void)threads;
  if (!reg || reg->kind == ORA_REG_NONE) return;  // regularizers.hpp:60
  const int64_t mn = m * n;
  if (reg->kind == ORA_REG_QUAD) {  // regularizers.cpp:53-55: V /= 1 + rho*alpha
    const double d = 1.0 + rho * reg->param;
#pragma omp parallel for num_threads(threads) schedule(static) if (threads > 1)
    for (int64_t t = 0; t < mn; ++t) V[t] /= d;
    return;
  }
  // regularizers.cpp:85-99: block soft-threshold at rho*lambda, group by group.
  const double thr = rho * reg->param;
#pragma omp parallel for num_threads(threads) schedule(dynamic, 64) if (threads > 1)
  for (int64_t g = 0; g < reg->num_groups; ++g) {
    double sq = 0.0;
    for (int64_t t = reg->offsets[g]; t < reg->offsets[g + 1]; ++t) {
      const double v = V[reg->cells[2 * t] * n + reg->cells[2 * t + 1]];
      sq += v * v;
    }
    const double nrm = std::sqrt(sq);
    if (nrm <= thr) {
      for (int64_t t = reg->offsets[g]; t < reg->offsets[g + 1]; ++t)
        V[reg->cells[2 * t] * n + reg->cells[2 * t + 1]] = 0.0;
    } else {
      const double scale = 1.0 - thr / nrm;
      for (int64_t t = reg->offsets[g]; t < reg->offsets[g + 1]; ++t)
        V[reg->cells[2 * t] * n + reg->cells[2 * t + 1]] *= scale;
    }
  }
}

double sq_norm(const double* v, int64_t len) {
  double s = 0.0;
  for (int64_t t = 0; t < len; ++t) s += v[t] * v[t];
  return s;
}

double reg_value(const ora_reg* reg, int64_t m, int64_t n, const double* X) {
  if (!reg || reg->kind == ORA_REG_NONE) return 0.0;
  if (reg->kind == ORA_REG_QUAD)  // regularizers.cpp:49-51
    return 0.5 * reg->param * sq_norm(X, m * n);
  double total = 0.0;  // regularizers.cpp:75-83
  for (int64_t g = 0; g < reg->num_groups; ++g) {
    double sq = 0.0;
    for (int64_t t = reg->offsets[g]; t < reg->offsets[g + 1]; ++t) {
      const double x = X[reg->cells[2 * t] * n + reg->cells[2 * t + 1]];
      sq += x * x;
    }
    total += std::sqrt(sq);
  }
  return reg->param * total;
}

// X1 - p and X^T 1 - q (solver.cpp:26-27, :83-84); sequential sums.
void residuals(const ora_problem* pr, const double* X, double* r, double* s,
               int threads) {
  const int64_t m = pr->m, n = pr->n;
#pragma omp parallel for num_threads(threads) schedule(static) if (threads > 1)
  for (int64_t i = 0; i < m; ++i) {
    double acc = 0.0;
    const double* row = X + i * n;
    for (int64_t j = 0; j < n; ++j) acc += row[j];
    r[i] = acc - pr->p[i];
  }
  if (threads <= 1) {
    std::vector<double> col(static_cast<size_t>(n), 0.0);
    for (int64_t i = 0; i < m; ++i) {
      const double* row = X + i * n;
      for (int64_t j = 0; j < n; ++j) col[j] += row[j];
    }
    for (int64_t j = 0; j < n; ++j) s[j] = col[j] - pr->q[j];
    return;
  }
#ifdef _OPENMP
  // Column sums: each thread owns a contiguous column range (fixed order in i).
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t jb = 0; jb < n; jb += 256) {
    const int64_t je = std::min(n, jb + 256);
    double acc[256] = {0.0};
    for (int64_t i = 0; i < m; ++i) {
      const double* row = X + i * n;
      for (int64_t j = jb; j < je; ++j) acc[j - jb] += row[j];
    }
    for (int64_t j = jb; j < je; ++j) s[j] = acc[j - jb] - pr->q[j];
  }
#endif
}

// solver.cpp:28-37 given r, s already in place.
void recurrence_tail(ora_state* st) {
  const double m = static_cast<double>(st->m);
  const double n = static_cast<double>(st->n);
  double rsum = 0.0;
  for (int64_t i = 0; i < st->m; ++i) rsum += st->r[i];
  st->eta = rsum / (m + n);
  const double shift = 2.0 * st->eta - st->theta;
  for (int64_t i = 0; i < st->m; ++i) {
    st->phi[i] = ((st->a[i] - 2.0 * st->r[i]) + shift) / n;
    st->a[i] -= st->r[i];
  }
  for (int64_t j = 0; j < st->n; ++j) {
    st->psi[j] = ((st->b[j] - 2.0 * st->s[j]) + shift) / m;
    st->b[j] -= st->s[j];
  }
  st->theta -= st->eta;
  ++st->k;
}

// solver.cpp:97-99: X <- [((X - rho C) + phi_i) + psi_j]_+ (std::max NaN semantics).
inline double clamp0(double v) { return v < 0.0 ? 0.0 : v; }

void clamp_pass(ora_state* st, const ora_problem* pr, double rho, int threads) {
  const int64_t m = pr->m, n = pr->n;
#pragma omp parallel for num_threads(threads) schedule(static) if (threads > 1)
  for (int64_t i = 0; i < m; ++i) {
    double* x = st->X + i * n;
    const double* c = pr->C + i * n;
    const double ph = st->phi[i];
    for (int64_t j = 0; j < n; ++j) x[j] = clamp0(((x[j] - rho * c[j]) + ph) + st->psi[j]);
  }
}

double vec_norm(const double* v, int64_t len) { return std::sqrt(sq_norm(v, len)); }

int64_t support_size(const double* X, int64_t len) {
  int64_t c = 0;
  for (int64_t t = 0; t < len; ++t) c += X[t] > 0.0;
  return c;
}

}  // namespace

extern "C" {

// ------------------------------------------------------------------- rng.hpp
void* ora_rng_new(uint64_t seed) { return new Rng(seed); }
void ora_rng_free(void* h) { delete static_cast<Rng*>(h); }
double ora_rng_uniform01(void* h) { return static_cast<Rng*>(h)->uniform01(); }
double ora_rng_normal(void* h) { return static_cast<Rng*>(h)->normal(); }
uint64_t ora_rng_raw(void* h) { return static_cast<Rng*>(h)->eng(); }

// ------------------------------------------------------------ datagen.cpp:43-54
void ora_squared_distance_cost(int64_t m, int64_t n, int64_t d, const double* a,
                               const double* b, double* C) {
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double sq = 0.0;
      for (int64_t t = 0; t < d; ++t) {
        const double diff = a[i * d + t] - b[j * d + t];
        sq += diff * diff;
      }
      C[i * n + j] = 0.5 * sq;
    }
}

// ------------------------------------------------------------ problem.cpp:41-74
int ora_validate_problem(int64_t m, int64_t n, const double* C, double* p, double* q,
                         char* msg, int msglen) {
  if (m < 1 || n < 1) {
    set_msg(msg, msglen, "cost must be at least 1x1");
    return ORA_E_DIMENSION;
  }
  for (int64_t t = 0; t < m * n; ++t) {
    if (!(C[t] >= 0.0) || !std::isfinite(C[t])) {
      set_msg(msg, msglen, "cost(" + std::to_string(t / n) + "," + std::to_string(t % n) +
                               ") must be finite and >= 0, got " + std::to_string(C[t]));
      return ORA_E_NEGATIVE;
    }
  }
  double* vs[2] = {p, q};
  const int64_t lens[2] = {m, n};
  const char* names[2] = {"p", "q"};
  for (int w = 0; w < 2; ++w) {  // problem.cpp:13-29 check_marginal
    double sum = 0.0;
    for (int64_t t = 0; t < lens[w]; ++t) {
      if (!(vs[w][t] >= 0.0) || !std::isfinite(vs[w][t])) {
        set_msg(msg, msglen, std::string(names[w]) + "[" + std::to_string(t) +
                                 "] must be finite and >= 0, got " +
                                 std::to_string(vs[w][t]));
        return ORA_E_NEGATIVE;
      }
      sum += vs[w][t];
    }
    if (std::abs(sum - 1.0) > kMarginalRejectTol) {
      set_msg(msg, msglen, std::string(names[w]) + " sums to " + std::to_string(sum) +
                               ", more than 1e-6 away from 1");
      return ORA_E_MARGINAL;
    }
  }
  for (int w = 0; w < 2; ++w) {  // problem.cpp:31-34 renormalize
    double sum = 0.0;
    for (int64_t t = 0; t < lens[w]; ++t) sum += vs[w][t];
    if (std::abs(sum - 1.0) > kMarginalSkipTol)
      for (int64_t t = 0; t < lens[w]; ++t) vs[w][t] /= sum;
  }
  return ORA_OK;
}

int ora_normalize_cost(int64_t m, int64_t n, double* C, int* all_zero) {
  double mx = -std::numeric_limits<double>::infinity();
  for (int64_t t = 0; t < m * n; ++t) mx = std::max(mx, C[t]);
  const bool zero = !(mx > 0.0);
  if (all_zero) *all_zero = zero ? 1 : 0;
  if (!zero)
    for (int64_t t = 0; t < m * n; ++t) C[t] /= mx;
  return ORA_OK;
}

double ora_primal_objective(const ora_problem* pr, const double* X, const ora_reg* reg) {
  double lin = 0.0;  // problem.cpp:84
  for (int64_t t = 0; t < pr->m * pr->n; ++t) lin += pr->C[t] * X[t];
  return lin + reg_value(reg, pr->m, pr->n, X);
}

// ------------------------------------------------------------ datagen.cpp:21-65
void ora_gaussian_problem(int64_t m, int64_t n, uint64_t seed, double* C, double* p,
                          double* q, double* src_pts, double* tgt_pts) {
  Rng rng(seed);
  auto cloud = [&](int64_t count, double* pts) {  // datagen.cpp:21-35
    const double mean_x = 2.0 * rng.normal();
    const double mean_y = 2.0 * rng.normal();
    const double l00 = 0.6 + 0.4 * rng.uniform01();
    const double l10 = 0.4 * rng.normal();
    const double l11 = 0.6 + 0.4 * rng.uniform01();
    for (int64_t i = 0; i < count; ++i) {
      const double z0 = rng.normal();
      const double z1 = rng.normal();
      pts[2 * i] = mean_x + l00 * z0;
      pts[2 * i + 1] = mean_y + l10 * z0 + l11 * z1;
    }
  };
  cloud(m, src_pts);
  cloud(n, tgt_pts);
  ora_squared_distance_cost(m, n, 2, src_pts, tgt_pts, C);
  for (int64_t i = 0; i < m; ++i) p[i] = 1.0 / static_cast<double>(m);  // :37-39
  for (int64_t j = 0; j < n; ++j) q[j] = 1.0 / static_cast<double>(n);
  ora_validate_problem(m, n, C, p, q, nullptr, 0);
  ora_normalize_cost(m, n, C, nullptr);
}

// ------------------------------------------------------------ datagen.cpp:67-129
int ora_adaptation_problem(int64_t m, int64_t n, int classes, uint64_t seed,
                           int identity_map, double* C, double* p, double* q,
                           double* src_pts, double* tgt_pts, int32_t* src_labels,
                           int32_t* tgt_labels) {
  if (classes < 1) return ORA_E_INVALID_ARG;
  if (m < classes || n < classes) return ORA_E_INVALID_ARG;
  Rng rng(seed);
  std::vector<double> mx(static_cast<size_t>(classes)), my(static_cast<size_t>(classes));
  for (int c = 0; c < classes; ++c) {
    const double ang = 2.0 * kPi * c / classes;
    mx[c] = 3.0 * std::cos(ang);
    my[c] = 3.0 * std::sin(ang);
  }
  const double spread = 0.85;
  auto labeled = [&](int64_t count, double* pts, int32_t* lab) {
    int64_t at = 0;
    for (int c = 0; c < classes; ++c) {
      const int64_t share = count / classes + (c < count % classes ? 1 : 0);
      for (int64_t t = 0; t < share; ++t, ++at) {
        pts[2 * at] = mx[c] + spread * rng.normal();
        pts[2 * at + 1] = my[c] + spread * rng.normal();
        lab[at] = c;
      }
    }
  };
  labeled(m, src_pts, src_labels);
  labeled(n, tgt_pts, tgt_labels);
  if (!identity_map) {
    const double sign = rng.uniform01() < 0.5 ? -1.0 : 1.0;
    const double angle = sign * (44.0 + 4.0 * rng.uniform01()) * kPi / 180.0;
    const double scale = 0.98 + 0.04 * rng.uniform01();
    const double tx = 0.2 * rng.normal();
    const double ty = 0.2 * rng.normal();
    const double ca = scale * std::cos(angle), sa = scale * std::sin(angle);
    for (int64_t j = 0; j < n; ++j) {
      const double x = tgt_pts[2 * j], y = tgt_pts[2 * j + 1];
      tgt_pts[2 * j] = ca * x - sa * y + tx;
      tgt_pts[2 * j + 1] = sa * x + ca * y + ty;
    }
  }
  ora_squared_distance_cost(m, n, 2, src_pts, tgt_pts, C);
  for (int64_t i = 0; i < m; ++i) p[i] = 1.0 / static_cast<double>(m);
  for (int64_t j = 0; j < n; ++j) q[j] = 1.0 / static_cast<double>(n);
  ora_validate_problem(m, n, C, p, q, nullptr, 0);
  ora_normalize_cost(m, n, C, nullptr);
  return ORA_OK;
}

// ------------------------------------------------------------- groups.cpp:37-60
int ora_column_class_blocks(const int32_t* labels, int64_t m, int64_t n,
                            int32_t* cells_out, int64_t* offsets_out,
                            int64_t* num_groups_out) {
  if (m < 1 || n < 1) return ORA_E_INVALID_ARG;
  int32_t classes = 0;
  for (int64_t i = 0; i < m; ++i) {
    if (labels[i] < 0) return ORA_E_INVALID_ARG;
    classes = std::max(classes, labels[i] + 1);
  }
  int64_t g = 0, t = 0;
  offsets_out[0] = 0;
  for (int64_t j = 0; j < n; ++j)
    for (int32_t c = 0; c < classes; ++c) {
      const int64_t start = t;
      for (int64_t i = 0; i < m; ++i)
        if (labels[i] == c) {
          cells_out[2 * t] = static_cast<int32_t>(i);
          cells_out[2 * t + 1] = static_cast<int32_t>(j);
          ++t;
        }
      if (t > start) offsets_out[++g] = t;
    }
  *num_groups_out = g;
  return ORA_OK;
}

void ora_prox(const ora_reg* reg, int64_t m, int64_t n, double* V, double rho) {
  prox_in_place(reg, m, n, V, rho, 1);
}

double ora_reg_value(const ora_reg* reg, int64_t m, int64_t n, const double* X) {
  return reg_value(reg, m, n, X);
}

// ------------------------------------------------------------- solver.cpp:55-93
double ora_default_stepsize(int64_t m, int64_t n) {
  return 2.0 / static_cast<double>(m + n);
}

void ora_default_init(int64_t m, int64_t n, double* phi0, double* psi0) {
  const double mn = static_cast<double>(m + n);
  const double ph = (1.0 + static_cast<double>(m) / mn) / (3.0 * mn);
  const double ps = (1.0 + static_cast<double>(n) / mn) / (3.0 * mn);
  for (int64_t i = 0; i < m; ++i) phi0[i] = ph;
  for (int64_t j = 0; j < n; ++j) psi0[j] = ps;
}

int ora_make_state(const ora_problem* pr, const double* X0, const double* phi0,
                   const double* psi0, ora_state* st, char* msg, int msglen) {
  const int64_t m = pr->m, n = pr->n;
  if (st->m != m || st->n != n) {
    set_msg(msg, msglen, "warm start dimensions do not match the problem");
    return ORA_E_DIMENSION;
  }
  if (X0) {
    for (int64_t t = 0; t < m * n; ++t)
      if (!std::isfinite(X0[t]) || X0[t] < 0.0) {
        set_msg(msg, msglen, "warm-start plan must be finite and >= 0");
        return ORA_E_NEGATIVE;
      }
    std::memcpy(st->X, X0, sizeof(double) * static_cast<size_t>(m * n));
    std::memcpy(st->phi, phi0, sizeof(double) * static_cast<size_t>(m));
    std::memcpy(st->psi, psi0, sizeof(double) * static_cast<size_t>(n));
  } else {
    std::memset(st->X, 0, sizeof(double) * static_cast<size_t>(m * n));
    ora_default_init(m, n, st->phi, st->psi);
  }
  residuals(pr, st->X, st->r, st->s, 1);
  for (int64_t i = 0; i < m; ++i) st->a[i] = static_cast<double>(n) * st->phi[i] + st->r[i];
  for (int64_t j = 0; j < n; ++j) st->b[j] = static_cast<double>(m) * st->psi[j] + st->s[j];
  double tot = 0.0;
  for (int64_t t = 0; t < m * n; ++t) tot += st->X[t];
  st->theta = (tot - 1.0) / static_cast<double>(m + n);
  st->eta = 0.0;
  st->k = 0;
  return ORA_OK;
}

// solver.cpp:95-102
void ora_step(ora_state* st, const ora_problem* pr, const ora_reg* reg, double rho,
              int threads) {
  clamp_pass(st, pr, rho, threads);
  prox_in_place(reg, pr->m, pr->n, st->X, rho, threads);
  residuals(pr, st->X, st->r, st->s, threads);
  recurrence_tail(st);
}

// duality.cpp:9-24 (+ regularizers.cpp:28-37, :57-62)
void ora_duality_gap(const ora_problem* pr, const ora_reg* reg, const ora_state* st,
                     double rho, double* dual_value, double* gap, double* dual_residual) {
  const int64_t m = pr->m, n = pr->n;
  // U = [Xbar - X]_+ with Xbar the clamp pass at the current state.
  std::vector<double> U(static_cast<size_t>(m * n));
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      const int64_t t = i * n + j;
      const double xbar = clamp0(((st->X[t] - rho * pr->C[t]) + st->phi[i]) + st->psi[j]);
      U[t] = clamp0(xbar - st->X[t]);
    }
  const double primal = ora_primal_objective(pr, st->X, reg);
  double pphi = 0.0, qpsi = 0.0;
  for (int64_t i = 0; i < m; ++i) pphi += pr->p[i] * st->phi[i];
  for (int64_t j = 0; j < n; ++j) qpsi += pr->q[j] * st->psi[j];
  const double linear = (pphi + qpsi) / rho;
  double conj = 0.0, dres = 0.0;
  const int kind = reg ? reg->kind : ORA_REG_NONE;
  if (kind == ORA_REG_QUAD) {
    conj = sq_norm(U.data(), m * n) / (2.0 * reg->param * rho * rho);
    dres = 0.0;
  } else {
    prox_in_place(reg, m, n, U.data(), 1.0, 1);
    dres = vec_norm(U.data(), m * n);
  }
  *dual_value = linear - conj;
  *gap = primal - *dual_value;
  *dual_residual = dres;
}

// solver.cpp:104-241
int ora_solve(const ora_problem* pr, const ora_reg* reg, const ora_options* opt,
              ora_state* st, ora_report* rep, ora_trace_row* trace, int64_t trace_cap,
              char* msg, int msglen) {
  if (opt->max_iter <= 0) {
    set_msg(msg, msglen, "max_iter must be positive, got " + std::to_string(opt->max_iter));
    return ORA_E_ZERO_ITERS;
  }
  if (opt->check_every <= 0) {
    set_msg(msg, msglen, "check_every must be positive");
    return ORA_E_INVALID_ARG;
  }
  if (!(opt->tol_primal > 0.0)) {
    set_msg(msg, msglen, "tol_primal must be positive");
    return ORA_E_INVALID_ARG;
  }
  if (opt->has_tol_gap && !(opt->tol_gap > 0.0)) {
    set_msg(msg, msglen, "tol_gap must be positive when set");
    return ORA_E_INVALID_ARG;
  }
  const int64_t m = pr->m, n = pr->n, mn = m * n;
  const int threads = opt->threads > 0 ? opt->threads : 1;
  const double rho = opt->rho > 0.0 ? opt->rho : ora_default_stepsize(m, n);
  rep->rho = rho;
  rep->trace_len = 0;
  rep->support_last_change = -1;

  std::vector<double> buf;  // fused path, solver.cpp:129-131
  bool shifted = false;
  if (opt->fused) buf.resize(static_cast<size_t>(mn));
  std::vector<char> mask;
  if (opt->record_trace) {
    mask.resize(static_cast<size_t>(mn));
    for (int64_t t = 0; t < mn; ++t) mask[t] = st->X[t] > 0.0;
    rep->support_last_change = 0;
  }
  const auto t0 = std::chrono::steady_clock::now();
  auto elapsed = [&] {
    if (opt->deterministic) return 0.0;
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
        .count();
  };
  double best = std::numeric_limits<double>::infinity();
  int64_t last_improvement = 0;
  rep->termination = ORA_TERM_MAXITER;

  for (int64_t k = 1; k <= opt->max_iter; ++k) {
    if (!opt->fused) {
      ora_step(st, pr, reg, rho, threads);
    } else {
      if (!shifted) {  // solver.cpp:161-168
        for (int64_t t = 0; t < mn; ++t) buf[t] = -rho * pr->C[t];
        for (int64_t i = 0; i < m; ++i)
          for (int64_t j = 0; j < n; ++j) {
            const int64_t t = i * n + j;
            st->X[t] = clamp0(((st->X[t] + buf[t]) + st->phi[i]) + st->psi[j]);
          }
        prox_in_place(reg, m, n, st->X, rho, threads);
        for (int64_t t = 0; t < mn; ++t) buf[t] += st->X[t];
        shifted = true;
      } else {  // solver.cpp:169-175
        for (int64_t i = 0; i < m; ++i)
          for (int64_t j = 0; j < n; ++j) {
            const int64_t t = i * n + j;
            st->X[t] = clamp0((buf[t] + st->phi[i]) + st->psi[j]);
          }
        prox_in_place(reg, m, n, st->X, rho, threads);
        shifted = false;
      }
      residuals(pr, st->X, st->r, st->s, threads);
      recurrence_tail(st);
    }

    const double r_primal = std::max(vec_norm(st->r, m), vec_norm(st->s, n));
    rep->r_primal = r_primal;
    if (!std::isfinite(r_primal)) {  // solver.cpp:181-185
      set_msg(msg, msglen, "non-finite iterate at iteration " + std::to_string(k) +
                               " (check rho and regularizer parameters)");
      rep->iterations = st->k;
      return ORA_E_NONFINITE;
    }
    if (opt->record_trace) {  // solver.cpp:187-198
      for (int64_t t = 0; t < mn; ++t) {
        const char on = st->X[t] > 0.0;
        if (mask[t] != on) {
          mask[t] = on;
          rep->support_last_change = k;
        }
      }
    }
    if (r_primal < best * (1.0 - kStallRelImprove)) {  // solver.cpp:200-203
      best = r_primal;
      last_improvement = k;
    }
    const bool at_check = (k % opt->check_every == 0);
    bool converged = false;
    double gap = std::numeric_limits<double>::quiet_NaN();
    double dres = std::numeric_limits<double>::quiet_NaN();
    const bool want_cert = (at_check && opt->has_tol_gap && r_primal <= opt->tol_primal) ||
                           (opt->record_trace && (at_check || k == opt->max_iter));
    if (want_cert) {
      double dv;
      ora_duality_gap(pr, reg, st, rho, &dv, &gap, &dres);
    }
    if (at_check && r_primal <= opt->tol_primal) {
      converged = !opt->has_tol_gap ||
                  (std::abs(gap) <= opt->tol_gap && dres <= opt->tol_gap);
    }
    if (opt->record_trace && (at_check || converged || k == opt->max_iter)) {
      if (rep->trace_len < trace_cap && trace) {
        ora_trace_row& row = trace[rep->trace_len];
        row.iter = k;
        row.r_primal = r_primal;
        row.gap = gap;
        row.dual_residual = dres;
        row.support = support_size(st->X, mn);
        row.elapsed_ms = elapsed();
      }
      ++rep->trace_len;
    }
    if (converged) {
      rep->termination = ORA_TERM_CONVERGED;
      break;
    }
    if (k - last_improvement >= kStallWindow) {
      rep->termination = ORA_TERM_STALLED;
      break;
    }
  }
  rep->iterations = st->k;
  rep->objective = ora_primal_objective(pr, st->X, reg);
  return ORA_OK;
}

// solver.cpp:243-256
int64_t ora_compute_skip_count(const ora_problem* pr) {
  const double m = static_cast<double>(pr->m);
  const double n = static_cast<double>(pr->n);
  double min_term = std::numeric_limits<double>::infinity();
  for (int64_t i = 0; i < pr->m; ++i)
    for (int64_t j = 0; j < pr->n; ++j) {
      const double denom = m * pr->p[i] + n * pr->q[j] + 1.0;
      const double term = std::ceil(pr->C[i * pr->n + j] * m * n / (m + n) / denom - 1.0);
      min_term = std::min(min_term, term);
    }
  return std::max<int64_t>(0, static_cast<int64_t>(min_term));
}

// tests/support/oracles.cpp:366-380 with the affine projection of
// oracles.cpp:16-37 written in closed form: z = w + u 1^T + 1 v^T,
// u_i = R_i/n - sum(R)/(n(m+n)), v_j = S_j/m - sum(S)/(m(m+n)),
// R = p - w1, S = q - w^T 1 (the minimum-norm solution of the rank-deficient
// normal equations; every solution gives the same z).
void ora_dr_reference(const ora_problem* pr, const ora_reg* reg, double rho,
                      const double* y0, int iters, double* xs, double* ys) {
  const int64_t m = pr->m, n = pr->n, mn = m * n;
  const double dm = static_cast<double>(m), dn = static_cast<double>(n);
  std::vector<double> y(y0, y0 + mn), x(static_cast<size_t>(mn)), w(static_cast<size_t>(mn));
  std::vector<double> R(static_cast<size_t>(m)), S(static_cast<size_t>(n));
  for (int it = 0; it < iters; ++it) {
    for (int64_t t = 0; t < mn; ++t) x[t] = clamp0(y[t] - rho * pr->C[t]);
    prox_in_place(reg, m, n, x.data(), rho, 1);
    for (int64_t t = 0; t < mn; ++t) w[t] = 2.0 * x[t] - y[t];
    double sR = 0.0, sS = 0.0;
    for (int64_t i = 0; i < m; ++i) {
      double acc = 0.0;
      for (int64_t j = 0; j < n; ++j) acc += w[i * n + j];
      R[i] = pr->p[i] - acc;
      sR += R[i];
    }
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int64_t i = 0; i < m; ++i) acc += w[i * n + j];
      S[j] = pr->q[j] - acc;
      sS += S[j];
    }
    for (int64_t i = 0; i < m; ++i) R[i] = R[i] / dn - sR / (dn * (dm + dn));
    for (int64_t j = 0; j < n; ++j) S[j] = S[j] / dm - sS / (dm * (dm + dn));
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j = 0; j < n; ++j) {
        const int64_t t = i * n + j;
        const double z = (w[t] + R[i]) + S[j];
        y[t] += z - x[t];
      }
    std::memcpy(xs + static_cast<size_t>(it) * mn, x.data(), sizeof(double) * mn);
    std::memcpy(ys + static_cast<size_t>(it) * mn, y.data(), sizeof(double) * mn);
  }
}

}  // extern "C"
