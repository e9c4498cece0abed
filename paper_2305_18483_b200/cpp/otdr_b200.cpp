// otdr_b200.cpp -- the reference's C++ solver API (include/otdr_b200/otdr.hpp)
// implemented on the C-ABI of include/otdr_dev.h. Host work here is the
// reference's setup logic (validation, partitions, option checks); every
// plan-sized pass runs in libotdr_dev.so on the GPU.
#include "otdr_b200/otdr.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <map>
#include <string>

#include "otdr_dev.h"

namespace otdr {

namespace {

constexpr double kMarginalRejectTol = 1e-6;  // problem.cpp:15
constexpr double kMarginalSkipTol = 1e-13;   // problem.cpp:18

[[noreturn]] void raise(otdr_status st, const std::string& msg) {
  switch (st) {
    case OTDR_E_DIMENSION: throw DimensionMismatch(msg);
    case OTDR_E_NEGATIVE: throw NegativeEntry(msg);
    case OTDR_E_MARGINAL: throw MarginalSumOutOfRange(msg);
    case OTDR_E_ZERO_ITERS: throw ZeroIterations(msg);
    case OTDR_E_INVALID_ARG: throw std::invalid_argument(msg);
    case OTDR_E_STATE: throw std::invalid_argument(msg);
    case OTDR_E_NONFINITE: throw NonFiniteIterate(msg);
    case OTDR_E_UNSUPPORTED: throw Unsupported(msg);
    default: throw DeviceError(msg.empty() ? "CUDA/NCCL failure" : msg);
  }
}

void check(otdr_dev* ctx, otdr_status st) {
  if (st != OTDR_OK) raise(st, ctx ? otdr_dev_last_error(ctx) : "");
}

void check_marginal(const Vector& v, const char* which) {  // problem.cpp:20-34
  for (Index i = 0; i < v.size(); ++i)
    if (!(v[i] >= 0.0) || !std::isfinite(v[i]))
      throw NegativeEntry(std::string(which) + "[" + std::to_string(i) +
                          "] must be finite and >= 0, got " + std::to_string(v[i]));
  const double s = v.sum();
  if (std::abs(s - 1.0) > kMarginalRejectTol)
    throw MarginalSumOutOfRange(std::string(which) + " sums to " + std::to_string(s) +
                                ", more than 1e-6 away from 1");
}

void renormalize(Vector& v) {
  const double s = v.sum();
  if (std::abs(s - 1.0) > kMarginalSkipTol)
    for (Index i = 0; i < v.size(); ++i) v[i] /= s;
}

char fmt_buf[64];
std::string with_param(const char* name, const char* key, double v) {
  std::snprintf(fmt_buf, sizeof(fmt_buf), "%s:%s=%g", name, key, v);
  return fmt_buf;
}

otdr_dev* open_context(const Problem& pr, Storage storage, int device) {
  otdr_dev_config cfg{};
  cfg.device = device;
  cfg.storage = storage == Storage::F64 ? OTDR_STORE_F64 : OTDR_STORE_F32;
  cfg.m = pr.rows();
  cfg.n = pr.cols();
  cfg.rank = 0;
  cfg.nranks = 1;
  cfg.row_begin = 0;
  cfg.row_end = pr.rows();
  otdr_dev* ctx = nullptr;
  const otdr_status st = otdr_dev_create(&cfg, &ctx);
  if (st != OTDR_OK) raise(st, "otdr_dev_create failed");
  const otdr_status up = otdr_dev_set_problem(ctx, pr.cost.data(), pr.p.data(), pr.q.data());
  if (up != OTDR_OK) {
    std::string msg = otdr_dev_last_error(ctx);
    otdr_dev_destroy(ctx);
    raise(up, msg);
  }
  return ctx;
}

void set_reg(otdr_dev* ctx, const Regularizer& reg, Index rows) {
  const int kind = reg.kind();
  if (kind != OTDR_REG_NONE && kind != OTDR_REG_QUAD && kind != OTDR_REG_GROUP_LASSO)
    throw Unsupported("regularizer " + reg.name() + " has no B200 kernel");
  std::vector<std::int32_t> labels;
  if (kind == OTDR_REG_GROUP_LASSO) labels = reg.row_labels(rows);
  check(ctx, otdr_dev_set_regularizer(ctx, static_cast<otdr_reg_kind>(kind), reg.param(),
                                      labels.empty() ? nullptr : labels.data()));
}

SolverState read_state(otdr_dev* ctx, Index m, Index n, bool with_plan) {
  SolverState st;
  if (with_plan) st.X = Matrix(m, n);
  st.phi = Vector(m);
  st.a = Vector(m);
  st.r = Vector(m);
  st.psi = Vector(n);
  st.b = Vector(n);
  st.s = Vector(n);
  int64_t k = 0;
  check(ctx, otdr_dev_get_state(ctx, with_plan ? st.X.data() : nullptr, st.phi.data(),
                                st.psi.data(), st.a.data(), st.b.data(), st.r.data(),
                                st.s.data(), &st.theta, &st.eta, &k));
  st.k = static_cast<long>(k);
  return st;
}

void write_state(otdr_dev* ctx, const SolverState& st, Index m, Index n) {
  if (st.X.rows() != m || st.X.cols() != n || st.phi.size() != m || st.psi.size() != n ||
      st.a.size() != m || st.b.size() != n || st.r.size() != m || st.s.size() != n)
    throw DimensionMismatch("solver state dimensions do not match the problem");
  check(ctx, otdr_dev_load_state(ctx, st.X.data(), st.phi.data(), st.psi.data(), st.a.data(),
                                 st.b.data(), st.r.data(), st.s.data(), st.theta, st.eta, st.k));
}

void set_init(otdr_dev* ctx, const std::optional<WarmStart>& init, Index m, Index n) {
  if (!init) {
    check(ctx, otdr_dev_set_state(ctx, nullptr, nullptr, nullptr));
    return;
  }
  const WarmStart& w = *init;
  if (w.plan0.rows() != m || w.plan0.cols() != n || w.phi0.size() != m || w.psi0.size() != n)
    throw DimensionMismatch("warm start dimensions do not match the problem");
  check(ctx, otdr_dev_set_state(ctx, w.plan0.data(), w.phi0.data(), w.psi0.data()));
}

struct Ctx {  // RAII for a one-call context
  otdr_dev* c;
  explicit Ctx(otdr_dev* x) : c(x) {}
  ~Ctx() { otdr_dev_destroy(c); }
};

SolveReport run_solve(otdr_dev* ctx, const SolverOptions& o, Index m, Index n, bool with_state) {
  otdr_solve_opts so{};
  so.rho = o.rho;
  so.max_iter = o.max_iter;
  so.tol_primal = o.tol_primal;
  so.has_tol_gap = o.tol_gap.has_value() ? 1 : 0;
  so.tol_gap = o.tol_gap.value_or(0.0);
  so.check_every = o.check_every;
  so.deterministic = o.deterministic ? 1 : 0;
  so.record_trace = o.record_trace ? 1 : 0;
  so.fused = o.fused ? 1 : 0;
  otdr_solve_result res{};
  check(ctx, otdr_dev_solve(ctx, &so, &res));
  SolveReport rep;
  rep.objective = res.objective;
  rep.iterations = static_cast<long>(res.iterations);
  rep.termination = static_cast<Termination>(res.termination);
  rep.rho = res.rho;
  rep.r_primal = res.r_primal;
  rep.support_last_change = static_cast<long>(res.support_last_change);
  rep.device_ms = res.device_ms;
  if (o.record_trace && res.trace_rows > 0) {
    std::vector<otdr_trace_row> rows(static_cast<std::size_t>(res.trace_rows));
    int64_t cnt = 0;
    check(ctx, otdr_dev_get_trace(ctx, rows.data(), res.trace_rows, &cnt));
    for (int64_t t = 0; t < cnt; ++t) {
      const auto& r = rows[static_cast<std::size_t>(t)];
      rep.trace.push_back(TraceRow{static_cast<long>(r.iter), r.r_primal, r.gap, r.dual_residual,
                                   static_cast<long>(r.support), r.elapsed_ms});
    }
  }
  if (with_state) rep.state = read_state(ctx, m, n, true);
  return rep;
}

void check_options(const SolverOptions& o) {  // solver.cpp:106-118
  if (o.max_iter <= 0)
    throw ZeroIterations("max_iter must be positive, got " + std::to_string(o.max_iter));
  if (o.check_every <= 0) throw std::invalid_argument("check_every must be positive");
  if (!(o.tol_primal > 0.0)) throw std::invalid_argument("tol_primal must be positive");
  if (o.tol_gap && !(*o.tol_gap > 0.0))
    throw std::invalid_argument("tol_gap must be positive when set");
}

}  // namespace

// ------------------------------------------------------------ problem.cpp
Problem validate_problem(Matrix cost, Vector p, Vector q) {
  if (cost.rows() < 1 || cost.cols() < 1) throw DimensionMismatch("cost must be at least 1x1");
  if (p.size() != cost.rows() || q.size() != cost.cols())
    throw DimensionMismatch("marginal lengths (" + std::to_string(p.size()) + ", " +
                            std::to_string(q.size()) + ") do not match cost " +
                            std::to_string(cost.rows()) + "x" + std::to_string(cost.cols()));
  for (Index i = 0; i < cost.rows(); ++i)
    for (Index j = 0; j < cost.cols(); ++j)
      if (!(cost(i, j) >= 0.0) || !std::isfinite(cost(i, j)))
        throw NegativeEntry("cost(" + std::to_string(i) + "," + std::to_string(j) +
                            ") must be finite and >= 0, got " + std::to_string(cost(i, j)));
  check_marginal(p, "p");
  check_marginal(q, "q");
  renormalize(p);
  renormalize(q);
  return Problem{std::move(cost), std::move(p), std::move(q)};
}

Problem normalize_cost(Problem problem, bool* all_zero) {
  double mx = -std::numeric_limits<double>::infinity();
  for (Index t = 0; t < problem.cost.size(); ++t) mx = std::max(mx, problem.cost.data()[t]);
  const bool zero = !(mx > 0.0);
  if (all_zero) *all_zero = zero;
  if (!zero)
    for (Index t = 0; t < problem.cost.size(); ++t) problem.cost.data()[t] /= mx;
  return problem;
}

double primal_objective(const Problem& problem, const Matrix& plan, const Regularizer& reg) {
  if (plan.rows() != problem.rows() || plan.cols() != problem.cols())
    throw DimensionMismatch("plan is " + std::to_string(plan.rows()) + "x" +
                            std::to_string(plan.cols()) + ", problem is " +
                            std::to_string(problem.rows()) + "x" + std::to_string(problem.cols()));
  Ctx ctx(open_context(problem, Storage::F64, 0));
  set_reg(ctx.c, reg, problem.rows());
  WarmStart w{plan, Vector(problem.rows()), Vector(problem.cols())};
  set_init(ctx.c, w, problem.rows(), problem.cols());
  double out = 0.0;
  check(ctx.c, otdr_dev_objective(ctx.c, &out));
  return out;
}

// -------------------------------------------------------------- groups.cpp
GroupPartition make_partition(Index rows, Index cols,
                              const std::vector<std::vector<GroupPartition::Cell>>& groups) {
  GroupPartition part;
  part.rows = rows;
  part.cols = cols;
  std::vector<char> seen(static_cast<std::size_t>(rows * cols), 0);
  for (const auto& grp : groups) {
    for (auto [i, j] : grp) {
      if (i < 0 || i >= rows || j < 0 || j >= cols)
        throw std::invalid_argument("group cell (" + std::to_string(i) + "," + std::to_string(j) +
                                    ") outside " + std::to_string(rows) + "x" +
                                    std::to_string(cols) + " grid");
      auto& s = seen[static_cast<std::size_t>(i) * static_cast<std::size_t>(cols) + j];
      if (s)
        throw std::invalid_argument("group cell (" + std::to_string(i) + "," + std::to_string(j) +
                                    ") appears in more than one group");
      s = 1;
      part.cells.emplace_back(i, j);
    }
    part.offsets.push_back(part.cells.size());
  }
  return part;
}

GroupPartition column_class_blocks(const std::vector<int>& row_labels, Index cols) {
  if (row_labels.empty()) throw std::invalid_argument("no row labels");
  if (cols < 1) throw std::invalid_argument("need at least one column");
  int classes = 0;
  for (int l : row_labels) {
    if (l < 0) throw std::invalid_argument("row labels must be >= 0");
    classes = std::max(classes, l + 1);
  }
  std::vector<std::vector<GroupPartition::Cell>> groups;
  for (Index j = 0; j < cols; ++j)
    for (int c = 0; c < classes; ++c) {
      std::vector<GroupPartition::Cell> cells;
      for (std::size_t i = 0; i < row_labels.size(); ++i)
        if (row_labels[i] == c)
          cells.emplace_back(static_cast<std::int32_t>(i), static_cast<std::int32_t>(j));
      if (!cells.empty()) groups.push_back(std::move(cells));
    }
  return make_partition(static_cast<Index>(row_labels.size()), cols, groups);
}

// -------------------------------------------------------- regularizers.cpp
QuadraticReg::QuadraticReg(double alpha) : alpha_(alpha) {
  if (!(alpha > 0.0) || !std::isfinite(alpha))
    throw std::invalid_argument("quadratic regularizer needs alpha > 0");
}
std::string QuadraticReg::name() const { return with_param("quad", "alpha", alpha_); }

GroupLassoReg::GroupLassoReg(double lambda, GroupPartition partition)
    : lambda_(lambda), partition_(std::move(partition)) {
  if (!(lambda > 0.0) || !std::isfinite(lambda))
    throw std::invalid_argument("group lasso needs lambda > 0");
}
std::string GroupLassoReg::name() const { return with_param("gl", "lambda", lambda_); }

// A partition maps onto the class-segment kernel when every group lies in one
// column and every column splits the covered rows into the same row sets
// (column_class_blocks, groups.cpp:37-60); row set order is irrelevant.
std::vector<std::int32_t> GroupLassoReg::row_labels(Index rows) const {
  if (partition_.rows != rows) throw DimensionMismatch("group partition rows do not match");
  const Index cols = partition_.cols;
  std::vector<std::int64_t> gid(static_cast<std::size_t>(rows * cols), -1);
  for (std::size_t g = 0; g < partition_.num_groups(); ++g) {
    const auto b = partition_.offsets[g], e = partition_.offsets[g + 1];
    for (auto t = b; t < e; ++t) {
      const auto [i, j] = partition_.cells[t];
      if (j != partition_.cells[b].second)
        throw Unsupported("group spans several columns: not a column_class_blocks partition");
      gid[static_cast<std::size_t>(i * cols + j)] = static_cast<std::int64_t>(g);
    }
  }
  std::vector<std::int32_t> label(static_cast<std::size_t>(rows), -1);
  std::map<std::int64_t, std::int32_t> canon;
  for (Index i = 0; i < rows; ++i) {
    const auto g = gid[static_cast<std::size_t>(i * cols)];
    if (g >= 0) {
      auto it = canon.find(g);
      if (it == canon.end()) it = canon.emplace(g, static_cast<std::int32_t>(canon.size())).first;
      label[static_cast<std::size_t>(i)] = it->second;
    }
  }
  for (Index j = 1; j < cols; ++j) {
    std::map<std::int64_t, std::int32_t> seen;
    std::map<std::int32_t, std::int64_t> back;
    for (Index i = 0; i < rows; ++i) {
      const auto g = gid[static_cast<std::size_t>(i * cols + j)];
      const auto l = label[static_cast<std::size_t>(i)];
      if ((g < 0) != (l < 0))
        throw Unsupported("columns cover different rows: not a column_class_blocks partition");
      if (g < 0) continue;
      auto [it, ins] = seen.emplace(g, l);
      auto [bt, bins] = back.emplace(l, g);
      if (it->second != l || bt->second != g)
        throw Unsupported("row sets differ across columns: not a column_class_blocks partition");
    }
  }
  return label;
}

// --------------------------------------------------------------- solver.cpp
const char* to_string(Termination t) {
  switch (t) {
    case Termination::Converged: return "Converged";
    case Termination::MaxIter: return "MaxIter";
    case Termination::Stalled: return "Stalled";
  }
  return "?";
}

double default_stepsize(Index m, Index n) { return 2.0 / static_cast<double>(m + n); }

WarmStart default_init(Index m, Index n) {
  const double mn = static_cast<double>(m + n);
  return WarmStart{Matrix::Zero(m, n),
                   Vector::Constant(m, (1.0 + static_cast<double>(m) / mn) / (3.0 * mn)),
                   Vector::Constant(n, (1.0 + static_cast<double>(n) / mn) / (3.0 * mn))};
}

SolverState make_state(const Problem& problem, const std::optional<WarmStart>& init) {
  Ctx ctx(open_context(problem, Storage::F64, 0));
  set_init(ctx.c, init, problem.rows(), problem.cols());
  return read_state(ctx.c, problem.rows(), problem.cols(), true);
}

void step(SolverState& state, const Problem& problem, const Regularizer& reg, double rho) {
  Ctx ctx(open_context(problem, Storage::F64, 0));
  set_reg(ctx.c, reg, problem.rows());
  write_state(ctx.c, state, problem.rows(), problem.cols());
  check(ctx.c, otdr_dev_step(ctx.c, rho, 1));
  state = read_state(ctx.c, problem.rows(), problem.cols(), true);
}

SolveReport solve(const Problem& problem, const Regularizer& reg, const SolverOptions& o) {
  check_options(o);
  Ctx ctx(open_context(problem, o.storage, o.device));
  set_reg(ctx.c, reg, problem.rows());
  set_init(ctx.c, o.init, problem.rows(), problem.cols());
  return run_solve(ctx.c, o, problem.rows(), problem.cols(), true);
}

long compute_skip_count(const Problem& pr, double /*rho*/) {  // solver.cpp:243-256
  const double m = static_cast<double>(pr.rows());
  const double n = static_cast<double>(pr.cols());
  double min_term = std::numeric_limits<double>::infinity();
  for (Index i = 0; i < pr.rows(); ++i)
    for (Index j = 0; j < pr.cols(); ++j) {
      const double denom = m * pr.p[i] + n * pr.q[j] + 1.0;
      min_term = std::min(min_term, std::ceil(pr.cost(i, j) * m * n / (m + n) / denom - 1.0));
    }
  return std::max(0L, static_cast<long>(min_term));
}

// -------------------------------------------------------------- duality.cpp
std::pair<Vector, Vector> recover_duals(const SolverState& state, double rho) {
  Vector mu(state.phi.size()), nu(state.psi.size());
  for (Index i = 0; i < mu.size(); ++i) mu[i] = state.phi[i] / rho;
  for (Index j = 0; j < nu.size(); ++j) nu[j] = state.psi[j] / rho;
  return {mu, nu};
}

DualCertificate duality_gap(const Problem& problem, const Regularizer& reg,
                            const SolverState& state, double rho) {
  Ctx ctx(open_context(problem, Storage::F64, 0));
  set_reg(ctx.c, reg, problem.rows());
  write_state(ctx.c, state, problem.rows(), problem.cols());
  otdr_certificate c{};
  check(ctx.c, otdr_dev_duality_gap(ctx.c, rho, &c));
  DualCertificate cert;
  std::tie(cert.mu, cert.nu) = recover_duals(state, rho);
  cert.dual_value = c.dual_value;
  cert.gap = c.gap;
  cert.dual_residual = c.dual_residual;
  return cert;
}

std::pair<double, Matrix> ot_cost_gradient(const Problem& problem, const Regularizer& reg,
                                           const SolverOptions& options) {
  SolveReport rep = solve(problem, reg, options);
  return {rep.objective, rep.plan()};
}

// ------------------------------------------------------------------ Session
namespace b200 {

Session::Session(const Problem& problem, const Regularizer& reg, Storage storage, int device)
    : m_(problem.rows()), n_(problem.cols()) {
  ctx_ = open_context(problem, storage, device);
  try {
    set_reg(ctx_, reg, m_);
  } catch (...) {
    otdr_dev_destroy(ctx_);
    throw;
  }
}
Session::~Session() { otdr_dev_destroy(ctx_); }
void Session::set_state(const std::optional<WarmStart>& init) { set_init(ctx_, init, m_, n_); }
void Session::load_state(const SolverState& st) { write_state(ctx_, st, m_, n_); }
void Session::step(double rho, long iters) { check(ctx_, otdr_dev_step(ctx_, rho, iters)); }
SolveReport Session::solve(const SolverOptions& o, bool with_state) {
  check_options(o);
  return run_solve(ctx_, o, m_, n_, with_state);
}
SolverState Session::state(bool with_plan) const { return read_state(ctx_, m_, n_, with_plan); }
double Session::objective() {
  double out = 0.0;
  check(ctx_, otdr_dev_objective(ctx_, &out));
  return out;
}
DualCertificate Session::duality_gap(double rho) {
  otdr_certificate c{};
  check(ctx_, otdr_dev_duality_gap(ctx_, rho, &c));
  DualCertificate cert;
  SolverState st = read_state(ctx_, m_, n_, false);
  std::tie(cert.mu, cert.nu) = recover_duals(st, rho);
  cert.dual_value = c.dual_value;
  cert.gap = c.gap;
  cert.dual_residual = c.dual_residual;
  return cert;
}

}  // namespace b200
}  // namespace otdr
