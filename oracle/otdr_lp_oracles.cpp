// otdr_lp_oracles.cpp -- algorithm-independent optimality oracles for the
// parity tests (TEST INFRASTRUCTURE ONLY; see otdr_oracle.h).
//
// The DR restatement in otdr_oracle.cpp checks the device iterates against the
// SAME algorithm; these oracles check converged plans against answers that do
// not come from Douglas-Rachford at all, as the reference's own suites do
// (proj/tests/support/oracles.cpp, used by proj/tests/test_solver.cpp:156-168
// and proj/tests/acceptance_main.cpp:186-244):
//
//   ora_affine_project    oracles.cpp:16-38   projection onto {X1 = p, X^T 1 = q}
//                                             (closed form of the rank-deficient
//                                             normal equations: any solution of the
//                                             consistent system gives the same X)
//   ora_polytope_project  oracles.cpp:44-71   Dykstra's alternating projections
//                                             onto the affine set and X >= 0
//   ora_projgrad_solve    oracles.cpp:73-101  argmin <C,X> + alpha/2 ||X||^2 over the
//                                             transport polytope: LP-vertex shortcut
//                                             with a linearized-optimality check,
//                                             else the projection of -C/alpha plus a
//                                             gradient-mapping certificate
//   ora_lp_vertex_solve   oracles.cpp:164-211 exact LP by enumerating spanning-tree
//                                             bases (m*n <= 12 or m, n <= 4)
//   ora_transport_simplex oracles.cpp:213-345 transportation simplex (north-west
//                                             corner start, Bland's rule)
//
// Plain dense row-major fp64 loops, compiled like the rest of the oracle.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <limits>
#include <numeric>
#include <utility>
#include <vector>

#include "otdr_oracle.h"

namespace {

constexpr double kFeasTol = 1e-9;  // oracles.cpp:13

using Mat = std::vector<double>;

// Z + u 1^T + 1 v^T with (u, v) solving n u + (1^T v) 1 = p - Z1,
// (1^T u) 1 + m v = q - Z^T 1.
void affine_project(int64_t m, int64_t n, const double* Z, const double* p, const double* q,
                    double* out) {
  const double dm = double(m), dn = double(n);
  std::vector<double> R(static_cast<size_t>(m)), S(static_cast<size_t>(n), 0.0);
  double sR = 0.0, sS = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    double acc = 0.0;
    for (int64_t j = 0; j < n; ++j) acc += Z[i * n + j];
    R[size_t(i)] = p[i] - acc;
    sR += R[size_t(i)];
  }
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) S[size_t(j)] += Z[i * n + j];
  for (int64_t j = 0; j < n; ++j) {
    S[size_t(j)] = q[j] - S[size_t(j)];
    sS += S[size_t(j)];
  }
  for (int64_t i = 0; i < m; ++i) R[size_t(i)] = R[size_t(i)] / dn - sR / (dn * (dm + dn));
  for (int64_t j = 0; j < n; ++j) S[size_t(j)] = S[size_t(j)] / dm - sS / (dm * (dm + dn));
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) out[i * n + j] = (Z[i * n + j] + R[size_t(i)]) + S[size_t(j)];
}

// Dykstra: x <- P_+(P_aff(x + ca) + cp), corrections ca, cp; stop when the
// marginals hold to tol AND the iterate stopped moving (oracles.cpp:57-66).
void polytope_project(int64_t m, int64_t n, const double* Z, const double* p, const double* q,
                      int max_iter, double tol, double* out) {
  const size_t mn = size_t(m * n);
  Mat x(Z, Z + mn), prev(Z, Z + mn), ca(mn, 0.0), cp(mn, 0.0), t(mn), y(mn);
  for (int it = 0; it < max_iter; ++it) {
    for (size_t k = 0; k < mn; ++k) t[k] = x[k] + ca[k];
    affine_project(m, n, t.data(), p, q, y.data());
    for (size_t k = 0; k < mn; ++k) ca[k] = t[k] - y[k];
    for (size_t k = 0; k < mn; ++k) {
      const double w = y[k] + cp[k];
      x[k] = w > 0.0 ? w : 0.0;
      cp[k] = w - x[k];
    }
    double viol = 0.0, change = 0.0, amax = 0.0;
    for (int64_t i = 0; i < m; ++i) {
      double acc = 0.0;
      for (int64_t j = 0; j < n; ++j) acc += x[size_t(i * n + j)];
      viol = std::max(viol, std::fabs(acc - p[i]));
    }
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int64_t i = 0; i < m; ++i) acc += x[size_t(i * n + j)];
      viol = std::max(viol, std::fabs(acc - q[j]));
    }
    for (size_t k = 0; k < mn; ++k) {
      change = std::max(change, std::fabs(x[k] - prev[k]));
      amax = std::max(amax, std::fabs(x[k]));
    }
    if (viol <= tol && change <= tol * (1.0 + amax)) break;
    prev = x;
  }
  std::memcpy(out, x.data(), mn * sizeof(double));
}

// Flow on a candidate basis by leaf peeling; false when the cells contain a
// cycle (not a spanning tree).
bool tree_flow(const std::vector<std::pair<int, int>>& cells, int m, int n, const double* p,
               const double* q, Mat& x) {
  const int nodes = m + n;
  std::vector<std::vector<int>> inc(static_cast<size_t>(nodes));
  for (int e = 0; e < int(cells.size()); ++e) {
    inc[size_t(cells[size_t(e)].first)].push_back(e);
    inc[size_t(m + cells[size_t(e)].second)].push_back(e);
  }
  std::vector<int> deg(static_cast<size_t>(nodes));
  std::vector<double> rem(static_cast<size_t>(nodes));
  for (int u = 0; u < nodes; ++u) deg[size_t(u)] = int(inc[size_t(u)].size());
  for (int i = 0; i < m; ++i) rem[size_t(i)] = p[i];
  for (int j = 0; j < n; ++j) rem[size_t(m + j)] = q[j];
  std::vector<char> used(cells.size(), 0);
  std::vector<double> flow(cells.size(), 0.0);
  std::deque<int> leaves;
  for (int u = 0; u < nodes; ++u)
    if (deg[size_t(u)] == 1) leaves.push_back(u);
  int solved = 0;
  while (!leaves.empty()) {
    const int u = leaves.front();
    leaves.pop_front();
    if (deg[size_t(u)] != 1) continue;
    int e = -1;
    for (int cand : inc[size_t(u)])
      if (!used[size_t(cand)]) {
        e = cand;
        break;
      }
    if (e < 0) continue;
    flow[size_t(e)] = rem[size_t(u)];
    used[size_t(e)] = 1;
    ++solved;
    const int other = cells[size_t(e)].first == u ? m + cells[size_t(e)].second : cells[size_t(e)].first;
    rem[size_t(other)] -= rem[size_t(u)];
    rem[size_t(u)] = 0.0;
    if (--deg[size_t(other)] == 1) leaves.push_back(other);
    deg[size_t(u)] = 0;
  }
  if (solved != int(cells.size())) return false;
  x.assign(size_t(m * n), 0.0);
  for (size_t e = 0; e < cells.size(); ++e) x[size_t(cells[e].first * n + cells[e].second)] = flow[e];
  return true;
}

int lp_vertex(int m, int n, const double* C, const double* p, const double* q, double* X,
              double* value) {
  if (!(m * n <= 12 || (m <= 4 && n <= 4))) return ORA_E_UNSUPPORTED;  // "TooLarge"
  double sp = 0.0, sq = 0.0;
  for (int i = 0; i < m; ++i) sp += p[i];
  for (int j = 0; j < n; ++j) sq += q[j];
  if (std::fabs(sp - sq) > kFeasTol) return ORA_E_MARGINAL;
  const int total = m * n, bs = m + n - 1;
  std::vector<int> pick(static_cast<size_t>(bs));
  std::iota(pick.begin(), pick.end(), 0);
  bool found = false;
  double best = 0.0;
  Mat x, bestx;
  for (;;) {
    std::vector<std::pair<int, int>> cells;
    for (int id : pick) cells.emplace_back(id / n, id % n);
    if (tree_flow(cells, m, n, p, q, x)) {
      const double lo = *std::min_element(x.begin(), x.end());
      if (lo >= -kFeasTol) {
        double val = 0.0;
        for (int k = 0; k < total; ++k) {
          x[size_t(k)] = x[size_t(k)] > 0.0 ? x[size_t(k)] : 0.0;
          val += x[size_t(k)] * C[k];
        }
        if (!found || val < best) {
          best = val;
          bestx = x;
          found = true;
        }
      }
    }
    int k = bs - 1;
    while (k >= 0 && pick[size_t(k)] == total - bs + k) --k;
    if (k < 0) break;
    ++pick[size_t(k)];
    for (int t = k + 1; t < bs; ++t) pick[size_t(t)] = pick[size_t(t - 1)] + 1;
  }
  if (!found) return ORA_E_INVALID_ARG;
  std::memcpy(X, bestx.data(), size_t(total) * sizeof(double));
  *value = best;
  return ORA_OK;
}

int simplex(int m, int n, const double* C, const double* p, const double* q, double* Xout,
            double* value) {
  double sp = 0.0, sq = 0.0;
  for (int i = 0; i < m; ++i) sp += p[i];
  for (int j = 0; j < n; ++j) sq += q[j];
  if (std::fabs(sp - sq) > kFeasTol) return ORA_E_MARGINAL;
  Mat x(static_cast<size_t>(m * n), 0.0);
  std::vector<char> basic(static_cast<size_t>(m * n), 0);
  auto X = [&](int i, int j) -> double& { return x[size_t(i * n + j)]; };
  auto B = [&](int i, int j) -> char& { return basic[size_t(i * n + j)]; };
  {  // north-west corner: one index advances per step -> m + n - 1 basic cells
    std::vector<double> pr(p, p + m), qr(q, q + n);
    int i = 0, j = 0;
    for (;;) {
      const double mv = std::min(pr[size_t(i)], qr[size_t(j)]);
      X(i, j) = mv;
      B(i, j) = 1;
      pr[size_t(i)] -= mv;
      qr[size_t(j)] -= mv;
      if (i == m - 1 && j == n - 1) break;
      if (pr[size_t(i)] <= qr[size_t(j)] && i < m - 1) ++i;
      else if (j < n - 1) ++j;
      else ++i;
    }
  }
  // path in the basis tree between nodes (rows 0..m-1, columns m..m+n-1)
  auto tree_path = [&](int from, int to, std::vector<int>& path) -> bool {
    std::vector<int> par(static_cast<size_t>(m + n), -2);
    std::deque<int> qu{from};
    par[size_t(from)] = -1;
    while (!qu.empty()) {
      const int u = qu.front();
      qu.pop_front();
      if (u == to) break;
      if (u < m) {
        for (int jj = 0; jj < n; ++jj)
          if (B(u, jj) && par[size_t(m + jj)] == -2) {
            par[size_t(m + jj)] = u;
            qu.push_back(m + jj);
          }
      } else {
        for (int ii = 0; ii < m; ++ii)
          if (B(ii, u - m) && par[size_t(ii)] == -2) {
            par[size_t(ii)] = u;
            qu.push_back(ii);
          }
      }
    }
    path.clear();
    for (int u = to; u != -1; u = par[size_t(u)]) {
      if (u == -2) return false;
      path.push_back(u);
    }
    std::reverse(path.begin(), path.end());
    return true;
  };
  std::vector<double> u(static_cast<size_t>(m)), v(static_cast<size_t>(n));
  std::vector<int> path;
  for (int pivot = 0; pivot < 100000; ++pivot) {
    // duals on the basis tree, u_0 = 0: c_ij = u_i + v_j on basic cells
    std::vector<char> known(static_cast<size_t>(m + n), 0);
    u[0] = 0.0;
    known[0] = 1;
    std::deque<int> qu{0};
    while (!qu.empty()) {
      const int node = qu.front();
      qu.pop_front();
      if (node < m) {
        for (int j = 0; j < n; ++j)
          if (B(node, j) && !known[size_t(m + j)]) {
            v[size_t(j)] = C[node * n + j] - u[size_t(node)];
            known[size_t(m + j)] = 1;
            qu.push_back(m + j);
          }
      } else {
        const int j = node - m;
        for (int i = 0; i < m; ++i)
          if (B(i, j) && !known[size_t(i)]) {
            u[size_t(i)] = C[i * n + j] - v[size_t(j)];
            known[size_t(i)] = 1;
            qu.push_back(i);
          }
      }
    }
    for (char k : known)
      if (!k) return ORA_E_INVALID_ARG;  // basis not spanning
    // Bland: first non-basic cell (row-major) with negative reduced cost
    int ei = -1, ej = -1;
    for (int i = 0; i < m && ei < 0; ++i)
      for (int j = 0; j < n; ++j)
        if (!B(i, j) && C[i * n + j] - u[size_t(i)] - v[size_t(j)] < -1e-10) {
          ei = i;
          ej = j;
          break;
        }
    if (ei < 0) {
      double val = 0.0;
      for (int k = 0; k < m * n; ++k) val += x[size_t(k)] * C[k];
      std::memcpy(Xout, x.data(), x.size() * sizeof(double));
      *value = val;
      return ORA_OK;
    }
    if (!tree_path(ei, m + ej, path)) return ORA_E_INVALID_ARG;
    // cycle: entering cell (+), then alternating along the tree path
    std::vector<std::pair<int, int>> cyc{{ei, ej}};
    for (size_t t = 0; t + 1 < path.size(); ++t) {
      const int a = path[t], b = path[t + 1];
      cyc.emplace_back(std::min(a, b), std::max(a, b) - m);
    }
    double th = std::numeric_limits<double>::infinity();
    size_t leave = 0;
    for (size_t t = 1; t < cyc.size(); t += 2) {
      const double f = X(cyc[t].first, cyc[t].second);
      if (f < th) {
        th = f;
        leave = t;
      }
    }
    for (size_t t = 0; t < cyc.size(); ++t) X(cyc[t].first, cyc[t].second) += (t % 2 == 0) ? th : -th;
    X(cyc[leave].first, cyc[leave].second) = 0.0;
    B(cyc[leave].first, cyc[leave].second) = 0;
    B(ei, ej) = 1;
  }
  return ORA_E_INVALID_ARG;  // pivot limit
}

}  // namespace

extern "C" {

void ora_affine_project(int64_t m, int64_t n, const double* Z, const double* p, const double* q,
                        double* out) {
  affine_project(m, n, Z, p, q, out);
}

void ora_polytope_project(int64_t m, int64_t n, const double* Z, const double* p, const double* q,
                          int max_iter, double tol, double* out) {
  polytope_project(m, n, Z, p, q, max_iter, tol, out);
}

int ora_lp_vertex_solve(int64_t m, int64_t n, const double* C, const double* p, const double* q,
                        double* X, double* value) {
  return lp_vertex(int(m), int(n), C, p, q, X, value);
}

int ora_transport_simplex(int64_t m, int64_t n, const double* C, const double* p,
                          const double* q, double* X, double* value) {
  return simplex(int(m), int(n), C, p, q, X, value);
}

// Returns ORA_OK with the plan in X, or ORA_E_NONFINITE when the gradient
// mapping certificate fails (the reference throws runtime_error); *gm gets
// the certificate value (0 on the LP-vertex shortcut).
int ora_projgrad_solve(int64_t m, int64_t n, const double* C, const double* p, const double* q,
                       double alpha, double* X, double* gm) {
  if (!(alpha > 0.0)) return ORA_E_INVALID_ARG;
  const size_t mn = size_t(m * n);
  *gm = 0.0;
  double cmax = 0.0;
  for (size_t k = 0; k < mn; ++k) cmax = std::max(cmax, std::fabs(C[k]));
  {
    // a vertex V is optimal iff it minimizes the linearized cost <C + alpha V, X>
    Mat V(mn), lin(mn), W(mn);
    double val = 0.0, rval = 0.0;
    if (simplex(int(m), int(n), C, p, q, V.data(), &val) == ORA_OK) {
      double lmax = 0.0, lv = 0.0;
      for (size_t k = 0; k < mn; ++k) {
        lin[k] = C[k] + alpha * V[k];
        lmax = std::max(lmax, std::fabs(lin[k]));
      }
      if (simplex(int(m), int(n), lin.data(), p, q, W.data(), &rval) == ORA_OK) {
        for (size_t k = 0; k < mn; ++k) lv += lin[k] * V[k];
        if (lv - rval <= 1e-11 * (1.0 + lmax)) {
          std::memcpy(X, V.data(), mn * sizeof(double));
          return ORA_OK;
        }
      }
    }
  }
  // <C,X> + alpha/2 ||X||^2 = alpha/2 ||X + C/alpha||^2 + const
  Mat z(mn), x(mn), st(mn), xs(mn);
  for (size_t k = 0; k < mn; ++k) z[k] = -C[k] / alpha;
  polytope_project(m, n, z.data(), p, q, 500000, 1e-13, x.data());
  const double t = 0.5 / alpha;
  for (size_t k = 0; k < mn; ++k) st[k] = x[k] - t * (C[k] + alpha * x[k]);
  polytope_project(m, n, st.data(), p, q, 500000, 1e-13, xs.data());
  double nrm = 0.0;
  for (size_t k = 0; k < mn; ++k) nrm += (x[k] - xs[k]) * (x[k] - xs[k]);
  *gm = std::sqrt(nrm) / t;
  std::memcpy(X, x.data(), mn * sizeof(double));
  return *gm > 1e-9 * (1.0 + cmax) ? ORA_E_NONFINITE : ORA_OK;
}

}  // extern "C"
