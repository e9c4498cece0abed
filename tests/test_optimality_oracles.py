"""Converged plans against algorithm-independent optimality oracles.

Every other parity test compares the device with a restatement of the SAME
Douglas-Rachford iteration. These compare converged device solves with answers
that do not come from DR at all -- the reference's own gates:

  * proj/tests/test_solver.cpp:156-168   strongly regularized 3x3 solve vs the
                                          projection oracle (plan <= 1e-5)
  * proj/tests/acceptance_main.cpp:186-211  criterion 1: 200 small unregularized
                                          problems vs exact LP vertex enumeration
                                          (|objective - LP| <= 1e-6)
  * acceptance_main.cpp:213-244          criterion 2: 100 seeds x alpha in
                                          {1e-3, 0.1, 1} quadratic vs
                                          projgrad_solve (plan <= 1e-5, value <= 1e-7)
  * acceptance_main.cpp:366-398          criterion 5: 200x300 gaussian problems,
                                          4 alphas x 10 seeds reach 1e-4 within
                                          50000 iterations (check_every 10)
  * acceptance_main.cpp:146-163, 460-471 criterion 8: the duality certificate of
                                          every converged run above has |gap| and
                                          dual residual <= 10 tol; unregularized
                                          runs satisfy LP complementary slackness
                                          and dual feasibility within 1e-5

The oracles (oracle/otdr_lp_oracles.cpp: transportation simplex, LP vertex
enumeration, Dykstra polytope projection, projgrad_solve) restate
proj/tests/support/oracles.cpp:16-345. The CPU tests pin them against the DR
oracle first (same gates, oracle on both sides); the GPU tests run the device
solve through the public API (otdr.solve, fp64 storage) and the device
certificate (otdr.duality_gap).
"""
import numpy as np
import pytest


class Certs:
    """acceptance_main.cpp:139-163 CertLog."""

    def __init__(self):
        self.gap = self.dres = self.cs = self.neg = 0.0
        self.runs = 0

    def add(self, cert_gap, cert_dres, tol, C=None, mu=None, nu=None, X=None):
        self.gap = max(self.gap, abs(cert_gap) / (10.0 * tol))
        self.dres = max(self.dres, cert_dres / (10.0 * tol))
        self.runs += 1
        if C is not None:
            slack = C - mu[:, None] - nu[None, :]
            self.neg = max(self.neg, float((-slack).max()))
            self.cs = max(self.cs, float(np.abs(X * slack).max()))

    def check(self, slackness):
        assert self.runs > 0
        assert self.gap <= 1.0 and self.dres <= 1.0, (self.gap, self.dres)
        if slackness:
            assert self.cs <= 1e-5 and self.neg <= 1e-5, (self.cs, self.neg)


# ---------------------------------------------------------------- CPU: pin the oracles
def test_oracle_projgrad_matches_dr_oracle(ora):
    """test_solver.cpp:156-168 with the DR oracle on the solver side."""
    C, p, q = ora.random_problem(ora.Rng(7), 3, 3)
    o = ora.solve(ora.Problem(C, p, q), ora.quad_reg(10.0), tol_primal=1e-9, tol_gap=1e-9,
                  max_iter=400000)
    assert o.termination == "Converged"
    assert np.abs(o.state.X - ora.projgrad_solve(C, p, q, 10.0)).max() <= 1e-5


def test_oracle_lp_enumeration_and_simplex_agree(ora):
    """Criterion 1 on the oracle: the two LP oracles agree, and the DR oracle
    reaches the LP value on all 200 small-suite problems."""
    worst = 0.0
    for sd in range(200):
        C, p, q = ora.small_suite_problem(sd)
        X1, v1 = ora.lp_vertex_solve(C, p, q)
        X2, v2 = ora.transport_simplex(C, p, q)
        assert abs(v1 - v2) <= 1e-12
        o = ora.solve(ora.Problem(C, p, q), ora.zero_reg(), tol_primal=1e-8, tol_gap=1e-7,
                      max_iter=1000000)
        assert o.termination == "Converged"
        worst = max(worst, abs(o.objective - v1))
    assert worst <= 1e-6


def test_oracle_projection_matches_dr_oracle(ora):
    """Criterion 2 on the oracle (DR oracle vs projgrad_solve)."""
    wp = wv = 0.0
    for sd in range(0, 100, 7):
        C, p, q = ora.random_problem(ora.Rng(4000 + sd), 3 if sd % 2 == 0 else 4, 3 if sd % 2 == 0 else 4)
        for a in (1e-3, 1e-1, 1.0):
            o = ora.solve(ora.Problem(C, p, q), ora.quad_reg(a), tol_primal=1e-12, tol_gap=1e-12,
                          max_iter=5000000)
            ref = ora.projgrad_solve(C, p, q, a)
            vref = float((C * ref).sum() + 0.5 * a * (ref * ref).sum())
            wp = max(wp, float(np.abs(o.state.X - ref).max()))
            wv = max(wv, abs(o.objective - vref))
    assert wp <= 1e-5 and wv <= 1e-7


def test_oracle_affine_and_polytope_projection(ora):
    """Projections land on the constraint sets; projecting a feasible point is
    the identity; the Dykstra projection beats random feasible points."""
    rng = np.random.default_rng(3)
    for m, n in ((3, 4), (5, 2), (6, 6)):
        p = rng.random(m) + 0.1
        q = rng.random(n) + 0.1
        p /= p.sum()
        q /= q.sum()
        Z = rng.normal(size=(m, n))
        A = ora.affine_project(Z, p, q)
        np.testing.assert_allclose(A.sum(axis=1), p, atol=1e-14)
        np.testing.assert_allclose(A.sum(axis=0), q, atol=1e-14)
        np.testing.assert_allclose(ora.affine_project(A, p, q), A, atol=1e-14)
        P = ora.polytope_project(Z, p, q)
        assert (P >= 0).all()
        np.testing.assert_allclose(P.sum(axis=1), p, atol=1e-11)
        np.testing.assert_allclose(P.sum(axis=0), q, atol=1e-11)
        d = float(((P - Z) ** 2).sum())
        for _ in range(50):  # random feasible points (plans of random couplings)
            F = np.outer(p, q) * (0.5 + rng.random((m, n)))
            F = ora.polytope_project(F, p, q)
            assert float(((F - Z) ** 2).sum()) >= d - 1e-12


# ---------------------------------------------------------------- GPU: device solves vs the oracles
gpu = pytest.mark.gpu


def _dev():
    return pytest.importorskip("paper_2305_18483_b200")


@gpu
def test_strongly_regularized_solve_matches_projection_oracle(ora):  # test_solver.cpp:156-168
    otdr = _dev()
    C, p, q = ora.random_problem(ora.Rng(7), 3, 3)
    pr = otdr.Problem(C, p, q)
    rep = otdr.solve(pr, otdr.QuadraticReg(10.0),
                     otdr.SolverOptions(tol_primal=1e-9, tol_gap=1e-9, max_iter=400000, storage="f64"))
    assert rep.termination.name == "Converged"
    ref = ora.projgrad_solve(C, p, q, 10.0)
    assert np.abs(rep.plan() - ref).max() <= 1e-5


@gpu
@pytest.mark.timeout(900, method="thread")
def test_acceptance_1_unregularized_vs_lp_and_certificates(ora):
    """acceptance_main.cpp:186-211 (+ criterion 8's slackness on these runs)."""
    otdr = _dev()
    certs = Certs()
    worst, converged = 0.0, 0
    opt = otdr.SolverOptions(tol_primal=1e-8, tol_gap=1e-7, max_iter=1000000, storage="f64")
    for sd in range(200):
        C, p, q = ora.small_suite_problem(sd)
        pr = otdr.Problem(C, p, q)
        rep = otdr.solve(pr, otdr.ZeroReg(), opt)
        if rep.termination.name != "Converged":
            continue
        converged += 1
        _, lpv = ora.lp_vertex_solve(C, p, q)
        worst = max(worst, abs(rep.objective - lpv))
        cert = otdr.duality_gap(pr, otdr.ZeroReg(), rep.state, rep.rho, storage="f64")
        certs.add(cert.gap, cert.dual_residual, opt.tol_primal, C, cert.mu, cert.nu, rep.plan())
    print(f"criterion 1: {converged}/200 converged, max |objective - LP| {worst:.2e}; "
          f"certs gap {certs.gap:.2f} dres {certs.dres:.2f} cs {certs.cs:.2e} neg {certs.neg:.2e}")
    assert converged == 200 and worst <= 1e-6
    certs.check(slackness=True)


@gpu
@pytest.mark.timeout(900, method="thread")
def test_acceptance_2_quadratic_vs_polytope_projection_and_certificates(ora):
    """acceptance_main.cpp:213-244 (+ criterion 8 on these runs)."""
    otdr = _dev()
    certs = Certs()
    wp = wv = 0.0
    converged = total = 0
    for sd in range(100):
        m = 3 if sd % 2 == 0 else 4
        C, p, q = ora.random_problem(ora.Rng(4000 + sd), m, m)
        pr = otdr.Problem(C, p, q)
        for a in (1e-3, 1e-1, 1.0):
            total += 1
            reg = otdr.QuadraticReg(a)
            opt = otdr.SolverOptions(tol_primal=1e-12, tol_gap=1e-12, max_iter=5000000, storage="f64")
            rep = otdr.solve(pr, reg, opt)
            if rep.termination.name != "Converged":
                continue
            converged += 1
            ref = ora.projgrad_solve(C, p, q, a)
            vref = float((C * ref).sum() + 0.5 * a * (ref * ref).sum())
            wp = max(wp, float(np.abs(rep.plan() - ref).max()))
            wv = max(wv, abs(rep.objective - vref))
            cert = otdr.duality_gap(pr, reg, rep.state, rep.rho, storage="f64")
            certs.add(cert.gap, cert.dual_residual, opt.tol_primal)
    print(f"criterion 2: {converged}/{total} converged, max plan diff {wp:.2e}, value diff {wv:.2e}; "
          f"certs gap {certs.gap:.2f} dres {certs.dres:.2f}")
    assert converged == total and wp <= 1e-5 and wv <= 1e-7
    certs.check(slackness=False)


@gpu
@pytest.mark.timeout(900, method="thread")
def test_acceptance_5_gaussian_200x300_in_budget_and_certificates(ora):
    """acceptance_main.cpp:366-398 (+ criterion 8 on these runs)."""
    otdr = _dev()
    certs = Certs()
    ok, worst_it = 0, 0
    for sd in range(10):
        C, p, q, *_ = ora.gaussian_problem(200, 300, sd)
        pr = otdr.Problem(C, p, q)
        for alpha in (5e-4, 5e-3, 5e-2, 2e-1):
            reg = otdr.QuadraticReg(alpha * 500.0)  # alpha scaled by m + n
            opt = otdr.SolverOptions(tol_primal=1e-4, max_iter=50000, check_every=10, storage="f64")
            rep = otdr.solve(pr, reg, opt)
            worst_it = max(worst_it, rep.iterations)
            if rep.termination.name == "Converged" and rep.r_primal <= 1e-4:
                ok += 1
                cert = otdr.duality_gap(pr, reg, rep.state, rep.rho, storage="f64")
                certs.add(cert.gap, cert.dual_residual, opt.tol_primal)
    print(f"criterion 5: {ok}/40 converged, max iterations {worst_it}; "
          f"certs gap {certs.gap:.2f} dres {certs.dres:.2f}")
    assert ok == 40
    certs.check(slackness=False)
