// otdr_b200/otdr.hpp -- the reference's C++ solver API on the B200 backend.
//
// Same names, argument meaning and exceptions as proj/include/otdr/
// {problem,groups,regularizers,solver,duality}.hpp. Every plan-sized operation
// runs on the GPU through the C-ABI of include/otdr_dev.h (libotdr_dev.so);
// this layer validates inputs and maps status codes back to exceptions.
#pragma once

#include <memory>
#include <optional>
#include <string>
#include <utility>
#include <vector>

#include "otdr_b200/errors.hpp"
#include "otdr_b200/types.hpp"

struct otdr_dev;

namespace otdr {

// ------------------------------------------------------------ problem.hpp
struct Problem {  // problem.hpp:13-21
  Matrix cost;
  Vector p, q;
  Index rows() const { return cost.rows(); }
  Index cols() const { return cost.cols(); }
};

class Regularizer;

Problem validate_problem(Matrix cost, Vector p, Vector q);         // problem.hpp:24
Problem normalize_cost(Problem problem, bool* all_zero = nullptr);  // problem.hpp:29
double primal_objective(const Problem& problem, const Matrix& plan,
                        const Regularizer& reg);                    // problem.hpp:32-33

// ------------------------------------------------------------- groups.hpp
struct GroupPartition {  // groups.hpp:15-27
  using Cell = std::pair<std::int32_t, std::int32_t>;
  Index rows = 0, cols = 0;
  std::vector<Cell> cells;
  std::vector<std::size_t> offsets{0};
  std::size_t num_groups() const { return offsets.size() - 1; }
  std::vector<Cell> group(std::size_t g) const {
    return {cells.begin() + static_cast<std::ptrdiff_t>(offsets[g]),
            cells.begin() + static_cast<std::ptrdiff_t>(offsets[g + 1])};
  }
};

GroupPartition make_partition(Index rows, Index cols,
                              const std::vector<std::vector<GroupPartition::Cell>>& groups);
GroupPartition column_class_blocks(const std::vector<int>& row_labels, Index cols);

// ------------------------------------------------------- regularizers.hpp
// The prox is applied inside the fused sweep kernel; the kind/parameter pair
// (and, for group lasso, the per-row class of a column_class_blocks-shaped
// partition) is what crosses the C-ABI.
class Regularizer {
 public:
  virtual ~Regularizer() = default;
  virtual std::string name() const = 0;
  virtual int kind() const = 0;       // otdr_reg_kind
  virtual double param() const = 0;
  // -1 = row in no group; throws Unsupported for partitions without a kernel.
  virtual std::vector<std::int32_t> row_labels(Index /*rows*/) const { return {}; }
};

class ZeroReg final : public Regularizer {  // regularizers.hpp:56-61
 public:
  std::string name() const override { return "none"; }
  int kind() const override { return 0; }
  double param() const override { return 0.0; }
};

class QuadraticReg final : public Regularizer {  // regularizers.hpp:63-79
 public:
  explicit QuadraticReg(double alpha);
  double alpha() const { return alpha_; }
  std::string name() const override;
  int kind() const override { return 1; }
  double param() const override { return alpha_; }

 private:
  double alpha_;
};

class GroupLassoReg final : public Regularizer {  // regularizers.hpp:81-96
 public:
  GroupLassoReg(double lambda, GroupPartition partition);
  double lambda() const { return lambda_; }
  const GroupPartition& partition() const { return partition_; }
  std::string name() const override;
  int kind() const override { return 2; }
  double param() const override { return lambda_; }
  std::vector<std::int32_t> row_labels(Index rows) const override;

 private:
  double lambda_;
  GroupPartition partition_;
};

// ------------------------------------------------------------- solver.hpp
enum class Storage { F32 = 0, F64 = 1 };

struct WarmStart {  // solver.hpp:34-37
  Matrix plan0;
  Vector phi0, psi0;
};

struct SolverOptions {  // solver.hpp:39-49 (+ storage / device)
  double rho = 0.0;
  long max_iter = 100000;
  double tol_primal = 1e-4;
  std::optional<double> tol_gap;
  long check_every = 1;
  bool deterministic = false;
  bool record_trace = false;
  bool fused = false;
  std::optional<WarmStart> init;
  Storage storage = Storage::F64;
  int device = 0;
};

struct SolverState {  // solver.hpp:51-59
  Matrix X;
  Vector phi, psi;
  Vector a, b;
  double theta = 0.0;
  Vector r, s;
  double eta = 0.0;
  long k = 0;
};

enum class Termination { Converged, MaxIter, Stalled };
const char* to_string(Termination t);

struct TraceRow {  // solver.hpp:65-72
  long iter;
  double r_primal;
  double gap;
  double dual_residual;
  long support;
  double elapsed_ms;
};

struct SolveReport {  // solver.hpp:74-87
  SolverState state;
  double objective = 0.0;
  long iterations = 0;
  Termination termination = Termination::MaxIter;
  double rho = 0.0;
  double r_primal = 0.0;
  std::vector<TraceRow> trace;
  long support_last_change = -1;
  double device_ms = 0.0;  // B200: device time of the iteration loop
  const Matrix& plan() const { return state.X; }
};

double default_stepsize(Index m, Index n);
WarmStart default_init(Index m, Index n);
SolverState make_state(const Problem& problem, const std::optional<WarmStart>& init);
void step(SolverState& state, const Problem& problem, const Regularizer& reg, double rho);
SolveReport solve(const Problem& problem, const Regularizer& reg, const SolverOptions& options);
long compute_skip_count(const Problem& problem, double rho);

// ------------------------------------------------------------ duality.hpp
struct DualCertificate {  // duality.hpp:19-24
  Vector mu, nu;
  double dual_value = 0.0;
  double gap = 0.0;
  double dual_residual = 0.0;
};
std::pair<Vector, Vector> recover_duals(const SolverState& state, double rho);
DualCertificate duality_gap(const Problem& problem, const Regularizer& reg,
                            const SolverState& state, double rho);
std::pair<double, Matrix> ot_cost_gradient(const Problem& problem, const Regularizer& reg,
                                           const SolverOptions& options);

// ------------------------------------------------------------ B200 session
namespace b200 {

// One device context holding C, X and the DR state in HBM for repeated steps
// and solves without re-uploading (the functions above create one per call).
class Session {
 public:
  Session(const Problem& problem, const Regularizer& reg, Storage storage = Storage::F64,
          int device = 0);
  ~Session();
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;

  void set_state(const std::optional<WarmStart>& init);
  void load_state(const SolverState& st);
  void step(double rho, long iters = 1);
  SolveReport solve(const SolverOptions& options, bool with_state = true);
  SolverState state(bool with_plan = true) const;
  double objective();
  DualCertificate duality_gap(double rho);

 private:
  otdr_dev* ctx_ = nullptr;
  Index m_, n_;
};

}  // namespace b200
}  // namespace otdr
