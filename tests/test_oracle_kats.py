"""Pins the CPU oracle against the reference's own known-answer tests.

The reference ships no golden files; its tests generate every input
from a seeded mt19937_64. Each case below restates one reference TEST_CASE
(file:line cited) against oracle/otdr_oracle.cpp, so the oracle is trusted before
the GPU path is checked against it.
"""
import math

import numpy as np
import pytest

pytestmark = []


def _zoo(ora, rng, m, n):
    """test_solver.cpp:31-47 -- the in-scope prefix of the regularizer zoo.

    Draws the WeightedL1 weights too so the warm-start draws that follow stay
    aligned with the reference's random stream."""
    labels = [i % 2 for i in range(m)]
    for _ in range(m * n):
        rng.uniform01()
    offs, cells = ora.column_class_blocks(labels, n)
    return [ora.zero_reg(), ora.quad_reg(0.7), ora.group_lasso_reg(0.02, offs, cells)]


def test_mt19937_64_known_answer(ora):
    # C++ [rand.predef]: the 10000th draw of a default-seeded mt19937_64.
    rng = ora.Rng(5489)
    for _ in range(9999):
        rng.raw()
    assert rng.raw() == 9981545732273789042


def test_default_stepsize_and_init(ora):  # test_solver.cpp:57-73
    assert ora.default_stepsize(2000, 3000) == pytest.approx(4e-4, rel=1e-15)
    assert ora.default_stepsize(1, 1) == 1.0
    assert ora.default_stepsize(1000, 1000) == pytest.approx(1e-3, rel=1e-15)
    X0, phi0, psi0 = ora.default_init(2, 3)
    assert not X0.any() and X0.shape == (2, 3)
    assert phi0[0] == pytest.approx(1.4 / 15.0, rel=1e-15) and phi0[1] == phi0[0]
    assert psi0[0] == pytest.approx(1.6 / 15.0, rel=1e-15) and psi0.shape == (3,)


def test_recurrence_matches_textbook_dr(ora):  # test_solver.cpp:75-116, acceptance :246-293
    worst = 0.0
    for seed in range(50):
        rng = ora.Rng(1000 + seed)
        m, n = 2 + seed % 5, 2 + (seed // 5) % 6
        C, p, q = ora.random_problem(rng, m, n)
        pr = ora.Problem(C, p, q)
        rho = ora.default_stepsize(m, n) if seed % 2 == 0 else 0.7 * ora.default_stepsize(m, n)
        for reg in _zoo(ora, rng, m, n):
            init = None
            if seed % 3 == 0:
                X0 = np.array([[0.3 * rng.uniform01() for _ in range(n)] for _ in range(m)])
                phi0 = np.array([rng.uniform01() - 0.5 for _ in range(m)])
                psi0 = np.array([rng.uniform01() - 0.5 for _ in range(n)])
                init = (X0, phi0, psi0)
            st = ora.make_state(pr, init)
            xs, ys = ora.dr_reference(pr, reg, rho, st.shadow(), 100)
            for t in range(100):
                ora.step(st, pr, reg, rho)
                worst = max(worst, np.abs(st.X - xs[t]).max(), np.abs(st.shadow() - ys[t]).max())
    assert worst <= 1e-9


def test_recurrence_tight_2x2(ora):  # test_solver.cpp:118-137
    C, p, q = ora.validate_problem([[0.0, 1.0], [1.0, 0.0]], [0.5, 0.5], [0.5, 0.5])
    pr = ora.Problem(C, p, q)
    rho = ora.default_stepsize(2, 2)
    st = ora.make_state(pr)
    reg = ora.zero_reg()
    _, ys = ora.dr_reference(pr, reg, rho, st.shadow(), 50)
    for t in range(50):
        ora.step(st, pr, reg, rho)
        assert np.abs(st.shadow() - ys[t]).max() <= 1e-10


def test_2x2_diagonal_plan(ora):  # test_solver.cpp:139-154
    pr = ora.Problem(*ora.validate_problem([[0.0, 1.0], [1.0, 0.0]], [0.5, 0.5], [0.5, 0.5]))
    rep = ora.solve(pr, ora.zero_reg(), tol_primal=1e-8)
    assert rep.termination == "Converged"
    assert np.abs(rep.state.X - np.diag([0.5, 0.5])).max() <= 1e-6
    assert abs(rep.objective) <= 1e-6


def test_1x1_all_regs_converge(ora):  # test_solver.cpp:170-192
    pr = ora.Problem(*ora.validate_problem([[0.8]], [1.0], [1.0]))
    offs = np.array([0, 1], dtype=np.int64)
    cells = np.array([[0, 0]], dtype=np.int32)
    for reg in (ora.zero_reg(), ora.quad_reg(3.0), ora.group_lasso_reg(2.0, offs, cells)):
        rep = ora.solve(pr, reg, tol_primal=1e-10, max_iter=200000)
        assert rep.termination == "Converged"
        assert abs(rep.state.X[0, 0] - 1.0) <= 1e-8


def test_skip_count_pins(ora):  # test_solver.cpp:194-237
    assert ora.compute_skip_count(ora.Problem(*ora.validate_problem([[1.0]], [1.0], [1.0]))) == 0
    n = 100
    big = ora.Problem(*ora.validate_problem(np.ones((n, n)), np.full(n, 1 / n), np.full(n, 1 / n)))
    assert ora.compute_skip_count(big) == 16
    wz = ora.Problem(*ora.validate_problem([[0.0, 1.0], [1.0, 2.0]], [0.5, 0.5], [0.5, 0.5]))
    assert ora.compute_skip_count(wz) == 0

    n = 20
    pr = ora.Problem(*ora.validate_problem(np.ones((n, n)), np.full(n, 1 / n), np.full(n, 1 / n)))
    rho = ora.default_stepsize(n, n)
    st = ora.make_state(pr, (np.outer(pr.p, pr.q), np.zeros(n), np.zeros(n)))
    zero_run = 0
    for k in range(1, 201):
        ora.step(st, pr, ora.zero_reg(), rho)
        if (st.X == 0.0).all():
            zero_run = k
        else:
            break
    assert zero_run == 19
    assert 0 <= ora.compute_skip_count(pr) <= zero_run


def test_row_col_residual_mass(ora):  # test_solver.cpp:239-249
    rng = ora.Rng(11)
    pr = ora.Problem(*ora.random_problem(rng, 5, 4))
    st = ora.make_state(pr)
    rho = ora.default_stepsize(5, 4)
    for _ in range(200):
        ora.step(st, pr, ora.quad_reg(0.3), rho)
        assert abs(st.r.sum() - st.s.sum()) <= 1e-10


def test_warm_restart_stationary(ora):  # test_solver.cpp:251-270
    rng = ora.Rng(13)
    pr = ora.Problem(*ora.random_problem(rng, 3, 3))
    reg = ora.quad_reg(0.5)
    rep = ora.solve(pr, reg, tol_primal=1e-10, max_iter=500000)
    assert rep.termination == "Converged"
    st = ora.make_state(pr, (rep.state.X, rep.state.phi, rep.state.psi))
    before = st.X.copy()
    ora.step(st, pr, reg, rep.rho)
    assert np.abs(st.X - before).max() <= 1e-8
    assert max(np.linalg.norm(st.r), np.linalg.norm(st.s)) <= 1e-8


def test_stall_window(ora):  # test_solver.cpp:272-286 (pinned-at-zero iterate)
    # The reference pins X at zero with a ForbiddenReg over every cell; a group
    # lasso whose single group per column is always annihilated does the same
    # with an in-scope regularizer.
    rng = ora.Rng(17)
    pr = ora.Problem(*ora.random_problem(rng, 3, 3))
    offs, cells = ora.column_class_blocks([0, 0, 0], 3)
    rep = ora.solve(pr, ora.group_lasso_reg(1e9, offs, cells), max_iter=30000)
    assert rep.termination == "Stalled"
    assert rep.iterations == 10001
    assert rep.r_primal > 0.1


def test_nonfinite_reported(ora):  # test_solver.cpp:288-301
    pr = ora.Problem(*ora.validate_problem([[0.1, 0.9]], [1.0], [0.5, 0.5]))
    with pytest.raises(ora.OracleError) as e:
        ora.solve(pr, ora.zero_reg(), init=(np.full((1, 2), 1e308), np.zeros(1), np.zeros(2)))
    assert e.value.code == ora.E_NONFINITE
    assert "non-finite iterate at iteration 1" in e.value.msg


def test_option_validation(ora):  # test_solver.cpp:303-340
    pr = ora.Problem(*ora.validate_problem([[0.0, 1.0], [1.0, 0.0]], [0.5, 0.5], [0.5, 0.5]))
    z = ora.zero_reg()
    for kw, code in [({"max_iter": 0}, ora.E_ZERO_ITERS), ({"max_iter": -5}, ora.E_ZERO_ITERS),
                     ({"check_every": 0}, ora.E_INVALID_ARG), ({"tol_primal": 0.0}, ora.E_INVALID_ARG),
                     ({"tol_gap": 0.0}, ora.E_INVALID_ARG)]:
        with pytest.raises(ora.OracleError) as e:
            ora.solve(pr, z, **kw)
        assert e.value.code == code
    with pytest.raises(ora.OracleError) as e:
        ora.solve(pr, z, init=(np.zeros((3, 2)), np.zeros(3), np.zeros(2)))
    assert e.value.code == ora.E_DIMENSION
    with pytest.raises(ora.OracleError) as e:
        ora.solve(pr, z, init=(np.full((2, 2), -0.1), np.zeros(2), np.zeros(2)))
    assert e.value.code == ora.E_NEGATIVE


def test_fused_matches_unfused(ora):  # test_solver.cpp:342-357
    rng = ora.Rng(19)
    for _ in range(5):
        pr = ora.Problem(*ora.random_problem(rng, 4, 5))
        a = ora.solve(pr, ora.quad_reg(0.4), max_iter=501, tol_primal=1e-300)
        b = ora.solve(pr, ora.quad_reg(0.4), max_iter=501, tol_primal=1e-300, fused=True)
        assert a.iterations == b.iterations == 501
        # X + (-rho C) == X - rho C exactly, so the even/odd path is bitwise equal.
        assert np.array_equal(a.state.X, b.state.X)
        assert np.array_equal(a.state.phi, b.state.phi)


def test_permutation_equivariance(ora):  # test_solver.cpp:359-391
    rng = ora.Rng(23)
    C, p, q = ora.random_problem(rng, 4, 5)
    sigma = [2, 0, 3, 1]
    tau = [4, 2, 0, 1, 3]
    Cp = C[np.ix_(sigma, tau)]
    pp, qp = p[sigma], q[tau]
    a = ora.solve(ora.Problem(C, p, q), ora.quad_reg(1.0), tol_primal=1e-9, max_iter=400000)
    b = ora.solve(ora.Problem(*ora.validate_problem(Cp, pp, qp)), ora.quad_reg(1.0), tol_primal=1e-9,
                  max_iter=400000)
    assert a.termination == b.termination == "Converged"
    assert np.abs(b.state.X - a.state.X[np.ix_(sigma, tau)]).max() <= 1e-6


def test_moderate_problems_converge(ora):  # test_solver.cpp:393-412
    rng = ora.Rng(29)
    n = 20
    pr = ora.Problem(*ora.random_problem(rng, n, n))
    offs, cells = ora.column_class_blocks([i % 4 for i in range(n)], n)
    for reg in (ora.zero_reg(), ora.quad_reg(0.05), ora.group_lasso_reg(0.01, offs, cells)):
        rep = ora.solve(pr, reg, tol_primal=1e-6, max_iter=200000)
        assert rep.termination == "Converged"
        assert rep.r_primal < 1e-6


def test_trace_support_settles(ora):  # test_solver.cpp:414-440
    rng = ora.Rng(41)
    pr = ora.Problem(*ora.random_problem(rng, 20, 20))
    rep = ora.solve(pr, ora.quad_reg(0.05), tol_primal=1e-7, max_iter=200000, record_trace=True,
                    check_every=10)
    assert rep.termination == "Converged" and rep.trace
    assert 0 <= rep.support_last_change < rep.iterations
    final_support = rep.trace[-1][4]
    for it, rp, gap, dres, support, _ in rep.trace:
        assert it % 10 == 0 and math.isfinite(gap) and math.isfinite(dres)
        if it > rep.support_last_change:
            assert support == final_support
    assert rep.trace[-1][1] <= 1e-7


def test_prox_pins(ora):  # test_regularizers.cpp:69-106, :135-149
    assert ora.prox(ora.quad_reg(1.0), [[1.0]], 1.0)[0, 0] == pytest.approx(0.5, rel=1e-15)
    whole = (np.array([0, 2], dtype=np.int64), np.array([[0, 0], [0, 1]], dtype=np.int32))
    out = ora.prox(ora.group_lasso_reg(2.5, *whole), [[3.0, 4.0]], 1.0)
    assert out[0, 0] == pytest.approx(1.5, rel=1e-14) and out[0, 1] == pytest.approx(2.0, rel=1e-14)
    assert ora.reg_value(ora.quad_reg(2.0), np.eye(2)) == pytest.approx(2.0, rel=1e-15)
    assert ora.reg_value(ora.group_lasso_reg(1.0, *whole), [[3.0, 4.0]]) == pytest.approx(5.0, rel=1e-15)
    offs, cells = ora.column_class_blocks([0, 0, 1, 1], 4)
    tiny = ora.prox(ora.group_lasso_reg(0.3, offs, cells), np.full((4, 4), 1e-3), 1.0)
    assert np.abs(tiny).max() == 0.0


def test_gl_prox_radial_oracle(ora):  # test_regularizers.cpp:135-149 (oracles.cpp:398-426)
    rng = ora.Rng(32)
    offs, cells = ora.column_class_blocks([0, 0, 1, 1], 4)
    reg = ora.group_lasso_reg(0.3, offs, cells)
    for rho in (0.05, 0.4, 1.0):
        v = np.array([[rng.uniform01() for _ in range(4)] for _ in range(4)])
        mine = ora.prox(reg, v, rho)
        for g in range(len(offs) - 1):
            idx = cells[offs[g]:offs[g + 1]]
            w = v[idx[:, 0], idx[:, 1]]
            nrm = np.linalg.norm(w)
            t = max(nrm - rho * 0.3, 0.0)  # argmin rho*lam*t + (t-|w|)^2/2 over t>=0
            np.testing.assert_allclose(mine[idx[:, 0], idx[:, 1]], w * (t / nrm), atol=1e-12)


def test_prox_preserves_zeros_nonneg(ora):  # test_regularizers.cpp:166-188
    rng = ora.Rng(34)
    offs, cells = ora.column_class_blocks([0, 0, 1, 1], 4)
    regs = [ora.zero_reg(), ora.quad_reg(0.8), ora.group_lasso_reg(0.3, offs, cells)]
    for _ in range(200):
        v = np.array([[rng.uniform01() for _ in range(4)] for _ in range(4)])
        v[np.array([[rng.uniform01() < 0.3 for _ in range(4)] for _ in range(4)])] = 0.0
        for reg in regs:
            out = ora.prox(reg, v, 0.2)
            assert not (out[v == 0.0] != 0.0).any()
            assert (out >= 0.0).all()


def test_problem_validation(ora):  # test_problem.cpp:30-105
    C, p, q = ora.validate_problem([[0.0]], [1.0], [1.0])
    assert p[0] == 1.0 and q[0] == 1.0
    c = [[0, 1], [1, 0]]
    for pp, qq in (([0.5, 0.6], [0.5, 0.5]), ([0.5, 0.5], [0.2, 0.2])):
        with pytest.raises(ora.OracleError) as e:
            ora.validate_problem(c, pp, qq)
        assert e.value.code == ora.E_MARGINAL
    _, p, q = ora.validate_problem(c, [0.5 + 4e-7, 0.5], [0.5, 0.5 - 4e-7])
    assert abs(p.sum() - 1) <= 1e-12 and abs(q.sum() - 1) <= 1e-12
    for args in (([[-1, 0], [0, 1]], [0.5, 0.5], [0.5, 0.5]), (c, [-0.1, 1.1], [0.5, 0.5]),
                 (c, [0.5, 0.5], [1.5, -0.5]), ([[0, np.inf], [1, 0]], [0.5, 0.5], [0.5, 0.5]),
                 (c, [np.nan, 1], [0.5, 0.5])):
        with pytest.raises(ora.OracleError) as e:
            ora.validate_problem(*args)
        assert e.value.code == ora.E_NEGATIVE
    for args in ((c, [1 / 3] * 3, [0.5, 0.5]), (c, [0.5, 0.5], [1 / 3] * 3)):
        with pytest.raises(ora.OracleError) as e:
            ora.validate_problem(*args)
        assert e.value.code == ora.E_DIMENSION
    _, p, q = ora.validate_problem(c, [1.0, 0.0], [0.0, 1.0])
    assert p[1] == 0.0 and q[0] == 0.0
    rng = ora.Rng(7)
    for _ in range(20):
        C = np.array([[rng.uniform01() for _ in range(4)] for _ in range(3)])
        p = np.array([rng.uniform01() + 0.05 for _ in range(3)])
        q = np.array([rng.uniform01() + 0.05 for _ in range(4)])
        p = p * ((1 + 3e-7) / p.sum())
        q = q * ((1 - 3e-7) / q.sum())
        once = ora.validate_problem(C, p, q)
        twice = ora.validate_problem(*once)
        for a, b in zip(once, twice):
            assert np.array_equal(a, b)


def test_normalize_cost_and_objective(ora):  # test_problem.cpp:107-216
    C, z = ora.normalize_cost([[2, 4], [1, 3]])
    assert np.array_equal(C, [[0.5, 1.0], [0.25, 0.75]]) and not z
    C, z = ora.normalize_cost([[0, 0], [0, 0]])
    assert z and not C.any()
    assert ora.normalize_cost([[1.0]])[0][0, 0] == 1.0
    pr = ora.Problem(*ora.validate_problem([[0, 1], [1, 0]], [0.5, 0.5], [0.5, 0.5]))
    assert ora.primal_objective(pr, np.diag([0.5, 0.5]), ora.zero_reg()) == 0.0
    one = ora.Problem(*ora.validate_problem([[1.0]], [1.0], [1.0]))
    assert ora.primal_objective(one, [[1.0]], ora.quad_reg(2.0)) == pytest.approx(2.0, rel=1e-15)


def test_column_class_blocks_order(ora):  # test_groups.cpp:54-86
    offs, cells = ora.column_class_blocks([0, 0, 0, 0], 3)
    assert len(offs) - 1 == 3
    for g in range(3):
        assert [tuple(c) for c in cells[offs[g]:offs[g + 1]]] == [(i, g) for i in range(4)]
    offs, cells = ora.column_class_blocks([0, 1, 0, 1], 3)
    assert len(offs) - 1 == 6 and all(offs[g + 1] - offs[g] == 2 for g in range(6))
    assert tuple(cells[offs[0]]) == (0, 0) and tuple(cells[offs[0] + 1]) == (2, 0)
    assert tuple(cells[offs[1]]) == (1, 0) and tuple(cells[offs[2]]) == (0, 1)
    offs, _ = ora.column_class_blocks([1, 0, 2, 1, 0], 4)
    assert offs[-1] == 20
    offs, _ = ora.column_class_blocks([0, 0, 3, 3], 2)
    assert len(offs) - 1 == 4
    with pytest.raises(ora.OracleError):
        ora.column_class_blocks([0, -1], 2)


def test_certificate_1x1(ora):  # test_duality.cpp:68-86
    pr = ora.Problem(*ora.validate_problem([[0.2]], [1.0], [1.0]))
    st = ora.make_state(pr, (np.ones((1, 1)), np.array([0.5]), np.array([0.25])))
    dv, gap, dres = ora.duality_gap(pr, ora.zero_reg(), st, 0.5)
    assert dv == pytest.approx(1.5, rel=1e-14)
    assert gap == pytest.approx(0.2 - 1.5, rel=1e-14)
    assert dres == pytest.approx(0.65, rel=1e-14)


def test_certificate_tight_2x2(ora):  # test_duality.cpp:99-108
    pr = ora.Problem(*ora.validate_problem([[0, 1], [1, 0]], [0.5, 0.5], [0.5, 0.5]))
    rep = ora.solve(pr, ora.zero_reg(), tol_primal=1e-8, tol_gap=1e-7, max_iter=500000)
    assert rep.termination == "Converged"
    _, gap, dres = ora.duality_gap(pr, ora.zero_reg(), rep.state, rep.rho)
    assert abs(gap) <= 1e-6 and dres <= 1e-6


def test_datagen_pins(ora):  # test_datagen.cpp:36-112
    C = ora.squared_distance_cost([[0, 0], [1, 0]], [[0, 1]])
    assert C[0, 0] == pytest.approx(0.5, rel=1e-15) and C[1, 0] == pytest.approx(1.0, rel=1e-15)
    C, p, q, src, tgt = ora.gaussian_problem(50, 60, 7)
    assert C.shape == (50, 60) and C.max() == 1.0 and C.min() >= 0.0
    assert np.abs(p - 0.02).max() <= 1e-15 and np.abs(q - 1 / 60).max() <= 1e-15
    C1, p1, *_ = ora.gaussian_problem(1, 1, 3)
    assert C1[0, 0] == 1.0 and p1[0] == 1.0
    a = ora.gaussian_problem(30, 40, 123)
    b = ora.gaussian_problem(30, 40, 123)
    c = ora.gaussian_problem(30, 40, 124)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    assert not np.array_equal(a[0], c[0])
    two = ora.adaptation_problem(4, 3, 2, 11)
    assert list(two[5]) == [0, 0, 1, 1]
    ap = ora.adaptation_problem(11, 7, 3, 21)
    assert list(np.bincount(ap[5])) == [4, 4, 3] and list(np.bincount(ap[6])) == [3, 2, 2]
    for args in ((4, 3, 0, 1), (2, 3, 3, 1)):
        with pytest.raises(ora.OracleError):
            ora.adaptation_problem(*args)


def test_identity_map_gl_purity(ora):  # test_datagen.cpp:115-124
    C, p, q, src, tgt, ls, lt = ora.adaptation_problem(20, 20, 2, 5, identity_map=True)
    offs, cells = ora.column_class_blocks(ls, 20)
    rep = ora.solve(ora.Problem(C, p, q), ora.group_lasso_reg(1e-3, offs, cells), tol_primal=1e-6,
                    max_iter=500000)
    assert rep.termination == "Converged"
    X = rep.state.X
    assert X[ls[:, None] == lt[None, :]].sum() / X.sum() >= 0.99


def test_acceptance_quadratic_sweeps(ora):  # acceptance_main.cpp:366-398 (criterion 5)
    worst = 0
    for sd in range(10):
        C, p, q, *_ = ora.gaussian_problem(200, 300, sd)
        pr = ora.Problem(C, p, q)
        for alpha in (5e-4, 5e-3, 5e-2, 2e-1):
            rep = ora.solve(pr, ora.quad_reg(alpha * 500.0), tol_primal=1e-4, max_iter=50000,
                            check_every=10)
            assert rep.termination == "Converged" and rep.r_primal <= 1e-4
            worst = max(worst, rep.iterations)
    assert worst <= 50000


def test_openmp_step_matches_single_thread(ora):
    """The threaded baseline sweep agrees with the faithful single-thread one."""
    C, p, q, *_ = ora.gaussian_problem(300, 517, 3)
    pr = ora.Problem(C, p, q)
    a = ora.make_state(pr)
    b = ora.make_state(pr)
    rho = ora.default_stepsize(300, 517)
    for _ in range(20):
        ora.step(a, pr, ora.quad_reg(5.0), rho, threads=1)
        ora.step(b, pr, ora.quad_reg(5.0), rho, threads=4)
    assert np.abs(a.X - b.X).max() <= 1e-13 * max(1.0, np.abs(a.X).max())
    assert np.array_equal(a.r, b.r)
