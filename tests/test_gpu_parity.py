"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle.

Gates (SURVEY §8(d) parity protocol; north-star tolerances):
  * fp64 storage: X, phi, psi after k in {1, 10, 100} steps within 1e-12 relative
    (max-norm) of the oracle -- element-wise arithmetic is the reference's, only
    the order of the row/column sums differs.
  * fp32 storage vs the oracle run on the fp32-rounded C: within 1e-5 relative.
  * solve(): same iteration count and termination as the oracle, objective and
    r_primal within 1e-6.
Plus the reference's own solver KATs re-run through the GPU-backed API.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

otdr = pytest.importorskip("paper_2305_18483_b200")


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def oracle_reg(ora, kind, param, labels, n):
    if kind == "none":
        return ora.zero_reg()
    if kind == "quad":
        return ora.quad_reg(param)
    offs, cells = ora.column_class_blocks(labels, n)
    return ora.group_lasso_reg(param, offs, cells)


def dev_reg(kind, param, labels, n):
    if kind == "none":
        return otdr.ZeroReg()
    if kind == "quad":
        return otdr.QuadraticReg(param)
    return otdr.GroupLassoReg(param, otdr.column_class_blocks(labels, n))


SHAPES = [(1, 1), (2, 2), (4, 5), (6, 7), (20, 20), (33, 257), (300, 517)]
REGS = [("none", 0.0), ("quad", 0.7), ("gl", 0.02)]


@pytest.mark.parametrize("m,n", SHAPES)
@pytest.mark.parametrize("kind,param", REGS)
def test_steps_fp64_match_oracle(ora, m, n, kind, param):
    C, p, q, *_ = ora.gaussian_problem(m, n, 5 + m)
    labels = [i % 3 for i in range(m)]
    pr = ora.Problem(C, p, q)
    oreg = oracle_reg(ora, kind, param, labels, n)
    st = ora.make_state(pr)
    eng = otdr.Engine(m, n, "f64")
    eng.set_problem(C, p, q)
    eng.set_regularizer(dev_reg(kind, param, labels, n))
    eng.set_state()
    rho = ora.default_stepsize(m, n)
    done = 0
    for k in (1, 10, 100):
        for _ in range(k - done):
            ora.step(st, pr, oreg, rho)
        eng.step(rho, k - done)
        done = k
        g = eng.get_state()
        assert g.k == st.k == k
        assert rel(g.X, st.X) <= 1e-12, (k, rel(g.X, st.X))
        assert rel(g.phi, st.phi) <= 1e-12
        assert rel(g.psi, st.psi) <= 1e-12
        assert rel(g.a, st.a) <= 1e-12 and rel(g.b, st.b) <= 1e-12
        assert abs(g.theta - st.theta) <= 1e-12 * max(1.0, abs(st.theta))


@pytest.mark.parametrize("m,n", [(6, 7), (300, 517), (1000, 1000)])
@pytest.mark.parametrize("kind,param", REGS)
def test_steps_fp32_match_oracle(ora, m, n, kind, param):
    C, p, q, *_ = ora.gaussian_problem(m, n, 11)
    C32 = C.astype(np.float32).astype(np.float64)  # same inputs on both sides
    labels = [i % 4 for i in range(m)]
    pr = ora.Problem(C32, p, q)
    oreg = oracle_reg(ora, kind, param * (m + n) if kind == "quad" else param, labels, n)
    st = ora.make_state(pr)
    eng = otdr.Engine(m, n, "f32")
    eng.set_problem(C, p, q)
    eng.set_regularizer(dev_reg(kind, param * (m + n) if kind == "quad" else param, labels, n))
    eng.set_state()
    rho = ora.default_stepsize(m, n)
    done = 0
    for k in (1, 10, 100):
        for _ in range(k - done):
            ora.step(st, pr, oreg, rho)
        eng.step(rho, k - done)
        done = k
        g = eng.get_state()
        assert rel(g.X, st.X) <= 1e-5, (k, rel(g.X, st.X))
        assert rel(g.phi, st.phi) <= 1e-5
        assert rel(g.psi, st.psi) <= 1e-5


def test_recurrence_matches_textbook_dr_on_gpu(ora):
    """test_solver.cpp:75-116 through the device step (warm starts, 0.7 rho)."""
    worst = 0.0
    for seed in range(0, 50, 3):
        rng = ora.Rng(1000 + seed)
        m, n = 2 + seed % 5, 2 + (seed // 5) % 6
        C, p, q = ora.random_problem(rng, m, n)
        pr = ora.Problem(C, p, q)
        rho = ora.default_stepsize(m, n) if seed % 2 == 0 else 0.7 * ora.default_stepsize(m, n)
        labels = [i % 2 for i in range(m)]
        for _ in range(m * n):
            rng.uniform01()
        for kind, param in (("none", 0.0), ("quad", 0.7), ("gl", 0.02)):
            init = None
            if seed % 3 == 0:
                X0 = np.array([[0.3 * rng.uniform01() for _ in range(n)] for _ in range(m)])
                phi0 = np.array([rng.uniform01() - 0.5 for _ in range(m)])
                psi0 = np.array([rng.uniform01() - 0.5 for _ in range(n)])
                init = (X0, phi0, psi0)
            ost = ora.make_state(pr, init)
            xs, ys = ora.dr_reference(pr, oracle_reg(ora, kind, param, labels, n), rho,
                                      ost.shadow(), 100)
            eng = otdr.Engine(m, n, "f64")
            eng.set_problem(C, p, q)
            eng.set_regularizer(dev_reg(kind, param, labels, n))
            eng.set_state(None if init is None else otdr.WarmStart(*init))
            for t in range(100):
                eng.step(rho, 1)
                g = eng.get_state()
                shadow = g.X + g.phi[:, None] + g.psi[None, :]
                worst = max(worst, np.abs(g.X - xs[t]).max(), np.abs(shadow - ys[t]).max())
    assert worst <= 1e-9


def _both_solve(ora, C, p, q, kind, param, labels, storage="f64", **kw):
    m, n = C.shape
    Co = C if storage == "f64" else C.astype(np.float32).astype(np.float64)
    orep = ora.solve(ora.Problem(Co, p, q), oracle_reg(ora, kind, param, labels, n), **kw)
    init = kw.pop("init", None)
    opts = otdr.SolverOptions(storage=storage, **{k: v for k, v in kw.items()})
    if init is not None:
        opts.init = otdr.WarmStart(*init)
    drep = otdr.solve(otdr.Problem(C, p, q), dev_reg(kind, param, labels, n), opts)
    return orep, drep


@pytest.mark.parametrize("kind,param", [("none", 0.0), ("quad", 0.05), ("gl", 0.01)])
def test_solve_matches_oracle_small(ora, kind, param):  # test_solver.cpp:393-412
    rng = ora.Rng(29)
    C, p, q = ora.random_problem(rng, 20, 20)
    labels = [i % 4 for i in range(20)]
    orep, drep = _both_solve(ora, C, p, q, kind, param, labels, tol_primal=1e-6, max_iter=200000)
    assert drep.termination.name == orep.termination == "Converged"
    assert drep.iterations == orep.iterations
    assert abs(drep.objective - orep.objective) <= 1e-6 * max(1.0, abs(orep.objective))
    assert abs(drep.r_primal - orep.r_primal) <= 1e-6
    assert rel(drep.plan(), orep.state.X) <= 1e-9


def test_solve_gaussian_1000_quad(ora):
    """cfg1: quadratic 1000^2, alpha = 5e-3 (m+n), tol 1e-4 -- both storages."""
    C, p, q, *_ = ora.gaussian_problem(1000, 1000, 0)
    for storage in ("f64", "f32"):
        orep, drep = _both_solve(ora, C, p, q, "quad", 10.0, None, storage=storage, tol_primal=1e-4)
        assert drep.termination.name == orep.termination == "Converged"
        if storage == "f64":
            assert drep.iterations == orep.iterations
        else:
            assert abs(drep.iterations - orep.iterations) <= max(2, orep.iterations // 100)
        assert abs(drep.objective - orep.objective) <= 1e-6 * abs(orep.objective)
        assert drep.r_primal <= 1e-4


def test_2x2_diagonal_and_1x1(ora):  # test_solver.cpp:139-154, :170-192
    pr = otdr.validate_problem([[0.0, 1.0], [1.0, 0.0]], [0.5, 0.5], [0.5, 0.5])
    rep = otdr.solve(pr, otdr.ZeroReg(), otdr.SolverOptions(tol_primal=1e-8))
    assert rep.termination == otdr.Termination.Converged
    assert np.abs(rep.plan() - np.diag([0.5, 0.5])).max() <= 1e-6
    assert abs(rep.objective) <= 1e-6
    one = otdr.validate_problem([[0.8]], [1.0], [1.0])
    for reg in (otdr.ZeroReg(), otdr.QuadraticReg(3.0),
                otdr.GroupLassoReg(2.0, otdr.make_partition(1, 1, [[(0, 0)]]))):
        rep = otdr.solve(one, reg, otdr.SolverOptions(tol_primal=1e-10, max_iter=200000))
        assert rep.termination == otdr.Termination.Converged
        assert abs(rep.plan()[0, 0] - 1.0) <= 1e-8


def test_stall_window_gpu(ora):  # test_solver.cpp:272-286
    rng = ora.Rng(17)
    C, p, q = ora.random_problem(rng, 3, 3)
    reg = otdr.GroupLassoReg(1e9, otdr.column_class_blocks([0, 0, 0], 3))
    rep = otdr.solve(otdr.Problem(C, p, q), reg, otdr.SolverOptions(max_iter=30000))
    assert rep.termination == otdr.Termination.Stalled
    assert rep.iterations == 10001
    assert rep.r_primal > 0.1


def test_nonfinite_and_options(ora):  # test_solver.cpp:288-340
    pr = otdr.validate_problem([[0.1, 0.9]], [1.0], [0.5, 0.5])
    with pytest.raises(otdr.NonFiniteIterate, match="non-finite iterate at iteration 1"):
        otdr.solve(pr, otdr.ZeroReg(), otdr.SolverOptions(
            init=otdr.WarmStart(np.full((1, 2), 1e308), np.zeros(1), np.zeros(2))))
    pr = otdr.validate_problem([[0.0, 1.0], [1.0, 0.0]], [0.5, 0.5], [0.5, 0.5])
    z = otdr.ZeroReg()
    with pytest.raises(otdr.ZeroIterations):
        otdr.solve(pr, z, otdr.SolverOptions(max_iter=0))
    with pytest.raises(ValueError):
        otdr.solve(pr, z, otdr.SolverOptions(check_every=0))
    with pytest.raises(ValueError):
        otdr.solve(pr, z, otdr.SolverOptions(tol_primal=0.0))
    with pytest.raises(ValueError):
        otdr.solve(pr, z, otdr.SolverOptions(tol_gap=0.0))
    with pytest.raises(otdr.DimensionMismatch):
        otdr.solve(pr, z, otdr.SolverOptions(init=otdr.WarmStart(np.zeros((3, 2)), np.zeros(3), np.zeros(2))))
    with pytest.raises(otdr.NegativeEntry):
        otdr.solve(pr, z, otdr.SolverOptions(init=otdr.WarmStart(np.full((2, 2), -0.1), np.zeros(2), np.zeros(2))))


@pytest.mark.parametrize("storage", ["f64", "f32"])
def test_fused_matches_unfused(ora, storage):  # test_solver.cpp:342-357
    rng = ora.Rng(19)
    for _ in range(3):
        C, p, q = ora.random_problem(rng, 4, 5)
        pr = otdr.Problem(C, p, q)
        a = otdr.solve(pr, otdr.QuadraticReg(0.4), otdr.SolverOptions(max_iter=501, tol_primal=1e-300, storage=storage))
        b = otdr.solve(pr, otdr.QuadraticReg(0.4), otdr.SolverOptions(max_iter=501, tol_primal=1e-300, fused=True, storage=storage))
        assert a.iterations == b.iterations == 501
        tol = 1e-12 if storage == "f64" else 1e-5
        assert rel(b.plan(), a.plan()) <= tol
        assert rel(b.state.phi, a.state.phi) <= tol


def test_trace_and_tol_gap(ora):  # test_solver.cpp:414-440, test_duality.cpp:99-108
    rng = ora.Rng(41)
    C, p, q = ora.random_problem(rng, 20, 20)
    orep, drep = _both_solve(ora, C, p, q, "quad", 0.05, None, tol_primal=1e-7, max_iter=200000,
                             record_trace=True, check_every=10, deterministic=True)
    assert drep.termination.name == "Converged" and drep.iterations == orep.iterations
    assert drep.support_last_change == orep.support_last_change
    assert len(drep.trace) == len(orep.trace)
    for dr, orow in zip(drep.trace, orep.trace):
        assert dr.iter == orow[0] and dr.support == orow[4]
        assert abs(dr.r_primal - orow[1]) <= 1e-9
        assert abs(dr.gap - orow[2]) <= 1e-8 and abs(dr.dual_residual - orow[3]) <= 1e-8
    pr = otdr.validate_problem([[0, 1], [1, 0]], [0.5, 0.5], [0.5, 0.5])
    rep = otdr.solve(pr, otdr.ZeroReg(), otdr.SolverOptions(tol_primal=1e-8, tol_gap=1e-7, max_iter=500000))
    o = ora.solve(ora.Problem(pr.cost, pr.p, pr.q), ora.zero_reg(), tol_primal=1e-8, tol_gap=1e-7, max_iter=500000)
    assert rep.termination.name == o.termination == "Converged"
    assert rep.iterations == o.iterations


def test_certificate_1x1():  # test_duality.cpp:68-86
    pr = otdr.validate_problem([[0.2]], [1.0], [1.0])
    st = otdr.make_state(pr, otdr.WarmStart(np.ones((1, 1)), np.array([0.5]), np.array([0.25])))
    cert = otdr.duality_gap(pr, otdr.ZeroReg(), st, 0.5)
    assert cert.mu[0] == pytest.approx(1.0, rel=1e-15) and cert.nu[0] == pytest.approx(0.5, rel=1e-15)
    assert cert.dual_value == pytest.approx(1.5, rel=1e-14)
    assert cert.gap == pytest.approx(0.2 - 1.5, rel=1e-14)
    assert cert.dual_residual == pytest.approx(0.65, rel=1e-14)


@pytest.mark.parametrize("kind,param", REGS)
def test_certificate_and_objective_match_oracle(ora, kind, param):
    C, p, q, *_ = ora.gaussian_problem(37, 45, 3)
    labels = [i % 3 for i in range(37)]
    pr = ora.Problem(C, p, q)
    st = ora.make_state(pr)
    oreg = oracle_reg(ora, kind, param, labels, 45)
    rho = ora.default_stepsize(37, 45)
    for _ in range(30):
        ora.step(st, pr, oreg, rho)
    dv, gap, dres = ora.duality_gap(pr, oreg, st, rho)
    dpr = otdr.Problem(C, p, q)
    dst = otdr.SolverState(st.X.copy(), st.phi.copy(), st.psi.copy(), st.a.copy(), st.b.copy(),
                           st.theta, st.r.copy(), st.s.copy(), st.eta, st.k)
    cert = otdr.duality_gap(dpr, dev_reg(kind, param, labels, 45), dst, rho)
    assert abs(cert.dual_value - dv) <= 1e-10 * max(1, abs(dv))
    assert abs(cert.gap - gap) <= 1e-10 * max(1, abs(gap))
    assert abs(cert.dual_residual - dres) <= 1e-10 * max(1, abs(dres))
    obj = otdr.primal_objective(dpr, st.X, dev_reg(kind, param, labels, 45))
    assert abs(obj - ora.primal_objective(pr, st.X, oreg)) <= 1e-12 * max(1, abs(obj))


def test_step_api_matches_oracle(ora):
    """make_state / step on host-visible states (value semantics)."""
    rng = ora.Rng(11)
    C, p, q = ora.random_problem(rng, 5, 4)
    pr = otdr.Problem(C, p, q)
    st = otdr.make_state(pr)
    ost = ora.make_state(ora.Problem(C, p, q))
    rho = otdr.default_stepsize(5, 4)
    for _ in range(50):
        otdr.step(st, pr, otdr.QuadraticReg(0.3), rho)
        ora.step(ost, ora.Problem(C, p, q), ora.quad_reg(0.3), rho)
        assert abs(st.r.sum() - st.s.sum()) <= 1e-10
    assert st.k == 50 and rel(st.X, ost.X) <= 1e-12


def test_gl_interleaved_and_uncovered_rows(ora):
    """Interleaved class labels (the test zoo's i%2) and a partition leaving a
    row uncovered map onto the class-sorted kernel exactly."""
    m, n = 9, 11
    C, p, q, *_ = ora.gaussian_problem(m, n, 8)
    groups = []
    rows_a = [0, 3, 6]
    rows_b = [1, 4, 7, 8]
    for j in range(n):
        groups.append([(i, j) for i in rows_a])
        groups.append([(i, j) for i in rows_b])
    part = otdr.make_partition(m, n, groups)
    offs = np.array([0] + list(np.cumsum([len(g) for g in groups])), dtype=np.int64)
    cells = np.array([c for g in groups for c in g], dtype=np.int32)
    oreg = ora.group_lasso_reg(0.004, offs, cells)
    pr = ora.Problem(C, p, q)
    st = ora.make_state(pr)
    eng = otdr.Engine(m, n, "f64")
    eng.set_problem(C, p, q)
    eng.set_regularizer(otdr.GroupLassoReg(0.004, part))
    eng.set_state()
    rho = ora.default_stepsize(m, n)
    for _ in range(40):
        ora.step(st, pr, oreg, rho)
    eng.step(rho, 40)
    g = eng.get_state()
    assert rel(g.X, st.X) <= 1e-12 and rel(g.phi, st.phi) <= 1e-12


@pytest.mark.parametrize("storage", ["f64", "f32"])
def test_device_cost_builder_matches_datagen(ora, storage):
    m, n = 123, 77
    C, p, q, src, tgt = ora.gaussian_problem(m, n, 9)
    eng = otdr.Engine(m, n, storage)
    zero = eng.build_sqdist_cost(src, tgt, p, q)
    assert not zero
    # the plan after one step from X = 0 exposes C through X1 = [phi+psi-rho C]_+
    eng.set_regularizer(otdr.ZeroReg())
    eng.set_state()
    rho = 0.25
    eng.step(rho, 1)
    g = eng.get_state()
    pr = ora.Problem(C if storage == "f64" else C.astype(np.float32).astype(np.float64), p, q)
    st = ora.make_state(pr)
    ora.step(st, pr, ora.zero_reg(), rho)
    if storage == "f64":
        assert np.array_equal(g.X, st.X)
    else:
        assert rel(g.X, st.X) <= 1e-6


def test_large_fp32_properties(ora):
    """Size-independent properties at 10000^2: mass balance sum r = sum s and
    non-negativity after several sweeps (cfg2 shape)."""
    m = n = 10000
    _, p, q, src, tgt = ora.gaussian_problem(8, 8, 0)
    rng = np.random.default_rng(0)
    src = rng.normal(size=(m, 2))
    tgt = rng.normal(size=(n, 2)) + 1.0
    p = np.full(m, 1.0 / m)
    q = np.full(n, 1.0 / n)
    eng = otdr.Engine(m, n, "f32")
    eng.build_sqdist_cost(src, tgt, p, q)
    eng.set_regularizer(otdr.ZeroReg())
    eng.set_state()
    eng.step(otdr.default_stepsize(m, n), 20)
    g = eng.get_state()
    assert g.k == 20
    assert (g.X >= 0).all()
    assert abs(g.r.sum() - g.s.sum()) <= 1e-9
    np.testing.assert_allclose(g.X.sum(axis=1) - p, g.r, atol=1e-9)


@pytest.mark.parametrize("kernel", ["auto", "twopass"])
@pytest.mark.parametrize("storage,m,n,classes", [
    ("f64", 3000, 300, 2),    # 1500-row class segments
    ("f32", 3000, 301, 2),
    ("f32", 1000, 1000, 10),  # the cfg3 shape at 1/10 scale
    ("f64", 2000, 203, 2),    # 1000-row segments
    ("f64", 4000, 64, 1),     # segment too long for the pipeline's staging: two-phase kernel
])
def test_gl_long_segments_match_oracle(ora, monkeypatch, kernel, storage, m, n, classes):
    if kernel != "auto":
        monkeypatch.setenv("OTDR_GL_KERNEL", kernel)
    C, p, q, src, tgt, ls, lt = ora.adaptation_problem(m, n, classes, 3)
    Co = C if storage == "f64" else C.astype(np.float32).astype(np.float64)
    pr = ora.Problem(Co, p, q)
    offs, cells = ora.column_class_blocks(ls, n)
    oreg = ora.group_lasso_reg(1e-3, offs, cells)
    st = ora.make_state(pr)
    eng = otdr.Engine(m, n, storage)
    eng.set_problem(C, p, q)
    eng.set_regularizer(otdr.GroupLassoReg(1e-3, otdr.column_class_blocks(ls, n)))
    eng.set_state()
    rho = ora.default_stepsize(m, n)
    for _ in range(12):
        ora.step(st, pr, oreg, rho)
    eng.step(rho, 12)
    g = eng.get_state()
    tol = 1e-12 if storage == "f64" else 1e-5
    assert rel(g.X, st.X) <= tol, rel(g.X, st.X)
    assert rel(g.phi, st.phi) <= tol and rel(g.psi, st.psi) <= tol


def test_gl_fused_and_trace_match_unfused(ora):
    C, p, q, src, tgt, ls, lt = ora.adaptation_problem(200, 150, 3, 5)
    pr = otdr.Problem(C, p, q)
    reg = otdr.GroupLassoReg(2e-3, otdr.column_class_blocks(ls, 150))
    a = otdr.solve(pr, reg, otdr.SolverOptions(max_iter=301, tol_primal=1e-300))
    b = otdr.solve(pr, reg, otdr.SolverOptions(max_iter=301, tol_primal=1e-300, fused=True))
    c = otdr.solve(pr, reg, otdr.SolverOptions(max_iter=301, tol_primal=1e-300, record_trace=True,
                                               check_every=50, deterministic=True))
    assert a.iterations == b.iterations == c.iterations == 301
    assert rel(b.plan(), a.plan()) <= 1e-12 and rel(c.plan(), a.plan()) <= 1e-12
    o = ora.solve(ora.Problem(C, p, q), ora.group_lasso_reg(2e-3, *ora.column_class_blocks(ls, 150)),
                  max_iter=301, tol_primal=1e-300, record_trace=True, check_every=50, deterministic=True)
    assert [r.support for r in c.trace] == [r[4] for r in o.trace]
    assert c.support_last_change == o.support_last_change


@pytest.mark.parametrize("storage", ["f64", "f32"])
@pytest.mark.parametrize("m,n,kind", [(20, 20, "none"), (300, 517, "quad"), (1000, 1000, "quad"),
                                      (5, 3000, "none"), (1500, 1400, "quad")])
def test_resident_matches_streaming(ora, monkeypatch, storage, m, n, kind):
    """The on-chip resident loop (grid mode) and the streaming graph loop give
    the same trajectory: fp64 storage -- same element-wise arithmetic,
    reduction order only; fp32 storage -- the resident loop runs on fp64
    shared-memory tiles (X rounded to fp32 only at write-back), so the two
    agree to the fp32 contract (1e-5)."""
    C, p, q, *_ = ora.gaussian_problem(m, n, 2)
    reg = otdr.QuadraticReg(5e-3 * (m + n)) if kind == "quad" else otdr.ZeroReg()
    out = {}
    for mode in ("on", "off"):
        monkeypatch.setenv("OTDR_RESIDENT", mode)
        eng = otdr.Engine(m, n, storage)
        eng.set_problem(C, p, q)
        eng.set_regularizer(reg)
        eng.set_state()
        eng.step(otdr.default_stepsize(m, n), 37)
        st = eng.get_state()
        eng.set_state()
        rep = eng.solve(otdr.SolverOptions(tol_primal=1e-6, max_iter=5000, storage=storage), with_state=True)
        out[mode] = (st, rep)
        eng.close()
    a, b = out["on"], out["off"]
    tol = 1e-12 if storage == "f64" else 1e-5
    assert a[0].k == b[0].k == 37
    assert rel(a[0].X, b[0].X) <= tol and rel(a[0].phi, b[0].phi) <= tol and rel(a[0].psi, b[0].psi) <= tol
    assert abs(a[0].theta - b[0].theta) <= (1e-12 if storage == "f64" else 1e-6) * max(1, abs(b[0].theta))
    assert a[1].termination == b[1].termination
    assert abs(a[1].iterations - b[1].iterations) <= (0 if storage == "f64" else 2)
    assert abs(a[1].objective - b[1].objective) <= (1e-9 if storage == "f64" else 1e-6) * abs(b[1].objective)


@pytest.mark.parametrize("mode", ["stream", "stream1", "resident"])
@pytest.mark.parametrize("storage", ["f64", "f32"])
def test_batched_solve_matches_sequential(ora, monkeypatch, storage, mode):
    """cfg5 shape at reduced batch: one launch (streaming with a 2-CTA cluster
    or one CTA per problem, or cluster-resident) == B solve()s."""
    monkeypatch.setenv("OTDR_BATCH", "resident" if mode == "resident" else "stream")
    if mode == "stream1":
        monkeypatch.setenv("OTDR_BATCH_CLUSTER", "1")
    B, m = 6, 96
    probs = [ora.gaussian_problem(m, m, b) for b in range(B)]
    alpha = 5e-3 * 2 * m
    reps = otdr.solve_batch([otdr.Problem(C, p, q) for (C, p, q, *_) in probs], otdr.QuadraticReg(alpha),
                            otdr.SolverOptions(tol_primal=1e-6, max_iter=20000, storage=storage))
    for (C, p, q, *_), rep in zip(probs, reps):
        Co = C if storage == "f64" else C.astype(np.float32).astype(np.float64)
        o = ora.solve(ora.Problem(Co, p, q), ora.quad_reg(alpha), tol_primal=1e-6, max_iter=20000)
        assert rep.termination.name == o.termination == "Converged"
        assert abs(rep.iterations - o.iterations) <= (0 if storage == "f64" else 3)
        assert abs(rep.objective - o.objective) <= 1e-6 * abs(o.objective)
        # the complete final state, as solve() returns it (solver.hpp:74-87)
        g, ost = rep.state, o.state
        assert g.k == rep.iterations
        if storage == "f64":
            for name in ("X", "phi", "psi", "a", "b"):
                assert rel(getattr(g, name), getattr(ost, name)) <= 1e-10, name
            # residuals r = X1 - p, s = X^T 1 - q cancel O(1/m) sums down to
            # O(tol): relative to themselves they carry ~1e-10 of summation order
            for name in ("r", "s"):
                assert rel(getattr(g, name), getattr(ost, name)) <= 1e-8, name
            assert abs(g.theta - ost.theta) <= 1e-12 * max(1.0, abs(ost.theta))
            # eta = sum(r)/(m+n) is a cancellation of O(1/m) residuals: absolute, like theta
            assert abs(g.eta - ost.eta) <= 1e-12
        else:
            assert rel(rep.plan(), ost.X) <= 1e-4
            assert rel(g.phi, ost.phi) <= 1e-4 and rel(g.psi, ost.psi) <= 1e-4
            assert np.isfinite(g.theta) and np.isfinite(g.eta)
            np.testing.assert_allclose(g.X.sum(axis=1) - p, g.r, atol=1e-7)
            np.testing.assert_allclose(g.X.sum(axis=0) - q, g.s, atol=1e-7)


@pytest.mark.parametrize("mode", ["stream", "resident"])
def test_batched_device_cost_and_512(ora, monkeypatch, mode):
    """512 x 512 per problem (the cfg5 tile): device-built costs, B = 3."""
    monkeypatch.setenv("OTDR_BATCH", mode)
    B, m = 3, 512
    src = np.empty((B, m, 2))
    tgt = np.empty((B, m, 2))
    ps = np.full((B, m), 1.0 / m)
    refs = []
    for b in range(B):
        C, p, q, s, t = ora.gaussian_problem(m, m, b)
        src[b], tgt[b] = s, t
        refs.append((C, p, q))
    be = otdr.BatchEngine(B, m, m, "f32")
    be.build_sqdist_costs(src, tgt, ps, ps)
    be.set_regularizer(otdr.QuadraticReg(5.12))
    reps = be.solve(otdr.SolverOptions(tol_primal=1e-4, max_iter=20000))
    X, phi, psi = be.plans()
    for b, (C, p, q) in enumerate(refs):
        o = ora.solve(ora.Problem(C.astype(np.float32).astype(np.float64), p, q), ora.quad_reg(5.12),
                      tol_primal=1e-4, max_iter=20000)
        assert reps[b].termination.name == "Converged"
        assert abs(reps[b].iterations - o.iterations) <= 3
        assert abs(reps[b].objective - o.objective) <= 1e-6 * abs(o.objective)


def test_batched_compressed_plans_bitwise(ora, monkeypatch):
    """B = 24 plans of 512^2 fp32 (24 MB, compressible by default; here also a
    4 MB compressible prefix) give bit-identical plans and reports to plain
    cudaMalloc plans."""
    B, m = 24, 512
    src = np.empty((B, m, 2))
    tgt = np.empty((B, m, 2))
    ps = np.full((B, m), 1.0 / m)
    for b in range(B):
        *_, s, t = ora.gaussian_problem(m, m, 100 + b)
        src[b], tgt[b] = s, t
    out = []
    for mode, cap in (("off", None), ("x", None), ("x", "0.004")):
        monkeypatch.setenv("OTDR_COMPRESS", mode)
        if cap:
            monkeypatch.setenv("OTDR_COMPRESS_GB", cap)
        else:
            monkeypatch.delenv("OTDR_COMPRESS_GB", raising=False)
        be = otdr.BatchEngine(B, m, m, "f32")
        be.build_sqdist_costs(src, tgt, ps, ps)
        be.set_regularizer(otdr.QuadraticReg(5.12))
        reps = be.solve(otdr.SolverOptions(tol_primal=1e-4, max_iter=20000))
        out.append(([(r.iterations, r.objective) for r in reps], be.plans()))
        be.close()
    for its, (X, phi, psi) in out[1:]:
        assert its == out[0][0]
        assert np.array_equal(X, out[0][1][0]) and np.array_equal(phi, out[0][1][1])
        assert np.array_equal(psi, out[0][1][2])


@pytest.mark.parametrize("kind", ["quad", "gl"])
def test_nccl_exchange_path_single_rank(ora, kind):
    """The row-sharded code path (reduce -> ncclAllReduce -> update, chunked
    host-polled graphs) on a 1-rank NCCL communicator equals the single-GPU path."""
    from paper_2305_18483_b200 import sharding
    m, n = 300, 257
    C, p, q, src, tgt, ls, lt = ora.adaptation_problem(m, n, 3, 1)
    reg = otdr.QuadraticReg(2.0) if kind == "quad" else otdr.GroupLassoReg(2e-3, otdr.column_class_blocks(ls, n))
    outs = []
    for shard in (None, otdr.Shard(0, 1, 0, m, sharding.nccl_unique_id())):
        eng = otdr.Engine(m, n, "f64", shard=shard)
        eng.set_problem(C, p, q)
        eng.set_regularizer(reg)
        eng.set_state()
        eng.step(otdr.default_stepsize(m, n), 25)
        st = eng.get_state()
        eng.set_state()
        rep = eng.solve(otdr.SolverOptions(tol_primal=1e-6, max_iter=5000))
        outs.append((st, rep))
        eng.close()
    (a, ra), (b, rb) = outs
    assert rel(a.X, b.X) <= 1e-12 and rel(a.phi, b.phi) <= 1e-12 and rel(a.psi, b.psi) <= 1e-12
    assert ra.termination == rb.termination and abs(ra.iterations - rb.iterations) <= 1
    assert abs(ra.objective - rb.objective) <= 1e-10 * abs(ra.objective)


@pytest.mark.parametrize("storage", ["f64", "f32"])
def test_otpb_device_io(ora, tmp_path, storage):
    """Cost read from an OTPB file straight into HBM, plan written back."""
    from paper_2305_18483_b200 import io
    m, n = 157, 211
    C, p, q, *_ = ora.gaussian_problem(m, n, 4)
    cpath, xpath = str(tmp_path / "c.otpb"), str(tmp_path / "x.otpb")
    io.write_matrix_otpb(cpath, C)
    eng = otdr.Engine(m, n, storage)
    eng.read_cost_otpb(cpath, p, q)
    eng.set_regularizer(otdr.QuadraticReg(1.5))
    eng.set_state()
    eng.step(otdr.default_stepsize(m, n), 30)
    eng.write_plan_otpb(xpath)
    st = eng.get_state()
    assert np.array_equal(io.read_matrix_otpb(xpath), st.X)
    ref = otdr.Engine(m, n, storage)
    ref.set_problem(C, p, q)
    ref.set_regularizer(otdr.QuadraticReg(1.5))
    ref.set_state()
    ref.step(otdr.default_stepsize(m, n), 30)
    assert np.array_equal(ref.get_state().X, st.X)
    io.write_matrix_otpb(cpath, C[:, :-1])
    with pytest.raises(otdr.DimensionMismatch):
        eng.read_cost_otpb(cpath, p, q)
    bad = C.copy()
    bad[3, 4] = -1.0
    io.write_matrix_otpb(cpath, bad)
    with pytest.raises(otdr.NegativeEntry):
        eng.read_cost_otpb(cpath, p, q)
    eng.close()
    ref.close()


@pytest.mark.parametrize("m,n", [(1, 1), (5, 3000), (33, 257), (300, 517), (1500, 1400), (2100, 700)])
@pytest.mark.parametrize("kind,param", [("none", 0.0), ("quad", 0.7)])
def test_stream_kernel_matches_oracle(ora, monkeypatch, m, n, kind, param):
    """The persistent streaming solve kernel (one cooperative launch for the
    whole solve / step run) against the oracle: fp64 iterates after k steps
    within 1e-12, then a full solve with the same iteration count."""
    monkeypatch.setenv("OTDR_RESIDENT", "off")
    C, p, q, *_ = ora.gaussian_problem(m, n, 17 + m)
    pr = ora.Problem(C, p, q)
    oreg = oracle_reg(ora, kind, param, None, n)
    st = ora.make_state(pr)
    eng = otdr.Engine(m, n, "f64")
    eng.set_problem(C, p, q)
    eng.set_regularizer(dev_reg(kind, param, None, n))
    eng.set_state()
    rho = ora.default_stepsize(m, n)
    done = 0
    for k in (1, 7, 40):
        for _ in range(k - done):
            ora.step(st, pr, oreg, rho)
        eng.step(rho, k - done)
        done = k
        g = eng.get_state()
        assert g.k == st.k == k
        assert rel(g.X, st.X) <= 1e-12, (k, rel(g.X, st.X))
        assert rel(g.phi, st.phi) <= 1e-12 and rel(g.psi, st.psi) <= 1e-12
        assert rel(g.a, st.a) <= 1e-12 and rel(g.b, st.b) <= 1e-12
        assert rel(g.r, st.r) <= 1e-9 and rel(g.s, st.s) <= 1e-9
        assert abs(g.theta - st.theta) <= 1e-12 * max(1.0, abs(st.theta))
    o = ora.solve(pr, oreg, tol_primal=1e-6, max_iter=3000)
    eng.set_state()
    rep = eng.solve(otdr.SolverOptions(tol_primal=1e-6, max_iter=3000, storage="f64"))
    assert rep.termination.name == o.termination
    assert rep.iterations == o.iterations
    assert abs(rep.objective - o.objective) <= 1e-9 * max(abs(o.objective), 1e-300)
    assert abs(rep.r_primal - o.r_primal) <= 1e-6
    eng.close()


@pytest.mark.parametrize("storage", ["f64", "f32"])
def test_stream_kernel_matches_graph_loop(ora, monkeypatch, storage):
    """Streaming kernel vs the three-kernel CUDA-graph loop on a plan larger
    than one wave: same trajectory (reduction order only)."""
    m, n = 3000, 2600
    C, p, q, *_ = ora.gaussian_problem(m, n, 3)
    out = {}
    for mode in ("on", "off"):
        monkeypatch.setenv("OTDR_RESIDENT", "off")
        monkeypatch.setenv("OTDR_STREAM", mode)
        eng = otdr.Engine(m, n, storage)
        eng.set_problem(C, p, q)
        eng.set_regularizer(otdr.QuadraticReg(5e-3 * (m + n)))
        eng.set_state()
        eng.step(otdr.default_stepsize(m, n), 25)
        st = eng.get_state()
        eng.set_state()
        rep = eng.solve(otdr.SolverOptions(tol_primal=1e-5, max_iter=5000, storage=storage))
        out[mode] = (st, rep)
        eng.close()
    a, b = out["on"], out["off"]
    tol = 1e-12 if storage == "f64" else 1e-6
    assert a[0].k == b[0].k == 25
    assert rel(a[0].X, b[0].X) <= tol and rel(a[0].phi, b[0].phi) <= tol and rel(a[0].psi, b[0].psi) <= tol
    assert a[1].termination == b[1].termination
    assert abs(a[1].iterations - b[1].iterations) <= (0 if storage == "f64" else 2)
    assert abs(a[1].objective - b[1].objective) <= (1e-9 if storage == "f64" else 1e-6) * abs(b[1].objective)


@pytest.mark.parametrize("storage", ["f64", "f32"])
def test_compressed_plan_is_bitwise_identical(ora, monkeypatch, storage):
    """X in a generically-compressible HBM allocation (default for plans
    >= 16 MB; here also split: first 4 MB compressible, rest plain, one
    contiguous range) gives the same iterates and solve, bit for bit, as a
    plain cudaMalloc plan -- compression is lossless, only traffic changes."""
    m, n = 2300, 2100
    C, p, q, *_ = ora.gaussian_problem(m, n, 12)
    out = {}
    for mode, cap in (("off", None), ("x", None), ("x", "0.004")):
        monkeypatch.setenv("OTDR_RESIDENT", "off")
        monkeypatch.setenv("OTDR_COMPRESS", mode)
        if cap:
            monkeypatch.setenv("OTDR_COMPRESS_GB", cap)
        else:
            monkeypatch.delenv("OTDR_COMPRESS_GB", raising=False)
        eng = otdr.Engine(m, n, storage)
        eng.set_problem(C, p, q)
        eng.set_regularizer(otdr.QuadraticReg(5e-3 * (m + n)))
        eng.set_state()
        eng.step(otdr.default_stepsize(m, n), 30)
        st = eng.get_state()
        eng.set_state()
        rep = eng.solve(otdr.SolverOptions(tol_primal=1e-5, max_iter=4000, storage=storage))
        out[(mode, cap)] = (st, rep)
        eng.close()
    base = out[("off", None)]
    for key in (("x", None), ("x", "0.004")):
        st, rep = out[key]
        assert np.array_equal(st.X, base[0].X) and np.array_equal(st.phi, base[0].phi), key
        assert np.array_equal(st.psi, base[0].psi) and st.theta == base[0].theta, key
        assert rep.iterations == base[1].iterations and rep.objective == base[1].objective, key


def _parallel(fns):
    """Run one callable per rank concurrently (ctypes releases the GIL), so
    every rank's exchange kernel is in flight at the same time."""
    import threading

    out, err = [None] * len(fns), []

    def run(i):
        try:
            out[i] = fns[i]()
        except BaseException as e:  # pragma: no cover - reported below
            err.append(e)

    th = [threading.Thread(target=run, args=(i,)) for i in range(len(fns))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in th), "a rank hung in the exchange"
    if err:
        raise err[0]
    return out


@pytest.mark.timeout(240, method="thread")  # a hung exchange must not hang the suite
@pytest.mark.parametrize("storage", ["f64", "f32"])
@pytest.mark.parametrize("world,kind", [(2, "quad"), (3, "none")])
def test_peer_exchange_ranks_on_one_gpu(ora, monkeypatch, storage, world, kind):
    """Row-sharded run with the in-kernel peer-memory exchange: `world` rank
    contexts on one GPU, linked in-process, each running the streaming kernel
    (grid capped so all ranks' kernels are co-resident). Iterates match the
    unsharded oracle; solve() stops at the same iteration on every rank."""
    monkeypatch.setenv("OTDR_STREAM_GRID", str(240 // world))
    from paper_2305_18483_b200 import sharding

    m, n = 900, 700
    C, p, q, *_ = ora.gaussian_problem(m, n, 31)
    Co = C if storage == "f64" else C.astype(np.float32).astype(np.float64)
    param = 5e-3 * (m + n) if kind == "quad" else 0.0
    pr = ora.Problem(Co, p, q)
    oreg = oracle_reg(ora, kind, param, None, n)
    st = ora.make_state(pr)
    bands = sharding.row_bands(m, world)
    engs = []
    for r, (lo, hi) in enumerate(bands):
        e = otdr.Engine(m, n, storage, shard=otdr.Shard(r, world, lo, hi, None))
        e.set_problem(C[lo:hi], p[lo:hi], q)
        e.set_regularizer(dev_reg(kind, param, None, n))
        engs.append(e)
    otdr.link_local(engs)
    assert all(e.solve_path() == "stream" for e in engs)
    _parallel([e.set_state for e in engs])
    rho = ora.default_stepsize(m, n)
    tol = 1e-12 if storage == "f64" else 1e-5
    done = 0
    for k in (1, 9, 30):
        for _ in range(k - done):
            ora.step(st, pr, oreg, rho)
        _parallel([lambda e=e: e.step(rho, k - done) for e in engs])
        done = k
        gs = _parallel([e.get_state for e in engs])
        X = np.concatenate([g.X for g in gs])
        phi = np.concatenate([g.phi for g in gs])
        assert rel(X, st.X) <= tol, (k, rel(X, st.X))
        assert rel(phi, st.phi) <= tol
        for g in gs:
            assert g.k == k
            assert rel(g.psi, st.psi) <= tol and rel(g.b, st.b) <= tol
            assert abs(g.theta - st.theta) <= (1e-12 if storage == "f64" else 1e-9) * max(1.0, abs(st.theta))
    _parallel([e.set_state for e in engs])
    o = ora.solve(pr, oreg, tol_primal=1e-6, max_iter=4000)
    reps = _parallel([lambda e=e: e.solve(otdr.SolverOptions(tol_primal=1e-6, max_iter=4000,
                                                             storage=storage), with_state=False)
                      for e in engs])
    for rep in reps:
        assert rep.termination.name == o.termination
        assert abs(rep.iterations - o.iterations) <= (0 if storage == "f64" else 2)
        assert abs(rep.r_primal - reps[0].r_primal) == 0.0
        assert abs(rep.objective - o.objective) <= (1e-9 if storage == "f64" else 1e-6) * abs(o.objective)
    for e in engs:
        e.close()


@pytest.mark.timeout(240, method="thread")  # a hung exchange must not hang the suite
@pytest.mark.parametrize("mode", ["stream", "graph"])
def test_peer_exchange_group_lasso(ora, monkeypatch, mode):
    """Group lasso on two rank contexts of one process, peers linked, no NCCL:
    the persistent GL solve kernel exchanges inside the kernel ("stream"), the
    graph loop through p2p_allreduce_kernel ("graph", OTDR_GL_STREAM=off).
    Bands are cut at class boundaries; iterates match the unsharded oracle.
    (The GL grid is capped so both ranks' persistent kernels are co-resident
    and a spinning exchange kernel never holds an SM the other rank needs --
    one GPU only.)"""
    monkeypatch.setenv("OTDR_GL_PIPE_GRID", "70")
    if mode == "graph":
        monkeypatch.setenv("OTDR_GL_STREAM", "off")
    from paper_2305_18483_b200 import sharding

    m, n, classes = 1200, 500, 4
    C, p, q, src, tgt, ls, lt = ora.adaptation_problem(m, n, classes, 5)
    pr = ora.Problem(C, p, q)
    offs, cells = ora.column_class_blocks(ls, n)
    oreg = ora.group_lasso_reg(2e-3, offs, cells)
    st = ora.make_state(pr)
    bands = sharding.row_bands(m, 2, ls)
    engs = []
    for r, (lo, hi) in enumerate(bands):
        e = otdr.Engine(m, n, "f64", shard=otdr.Shard(r, 2, lo, hi, None))
        e.set_problem(C[lo:hi], p[lo:hi], q)
        e.set_regularizer(otdr.GroupLassoReg(2e-3, otdr.column_class_blocks(ls, n)),
                          labels_local=np.asarray(ls)[lo:hi])
        engs.append(e)
    otdr.link_local(engs)
    assert all(e.solve_path() == mode for e in engs)
    _parallel([e.set_state for e in engs])
    rho = ora.default_stepsize(m, n)
    for _ in range(15):
        ora.step(st, pr, oreg, rho)
    _parallel([lambda e=e: e.step(rho, 15) for e in engs])
    gs = _parallel([e.get_state for e in engs])
    X = np.concatenate([g.X for g in gs])
    assert rel(X, st.X) <= 1e-12, rel(X, st.X)
    assert rel(np.concatenate([g.phi for g in gs]), st.phi) <= 1e-12
    assert all(rel(g.psi, st.psi) <= 1e-12 for g in gs)
    for e in engs:
        e.close()


def test_headline_size_stream_vs_graph_solve(monkeypatch):
    """The north-star point (20000^2, quadratic alpha = 200, fp32): a full solve
    to 1e-4 through the streaming kernel and through the CUDA-graph loop stop
    at the same iteration (+-2, fp32 reduction order) with the same objective
    (1e-6 relative) -- full-size parity between the two device loops."""
    from paper_2305_18483_b200 import datagen

    m = n = 20000
    src, tgt = datagen.gaussian_points(m, n, 0)
    out = {}
    for mode in ("on", "off"):
        monkeypatch.setenv("OTDR_STREAM", mode)
        eng = otdr.Engine(m, n, "f32")
        eng.build_sqdist_cost(src, tgt, datagen.uniform(m), datagen.uniform(n))
        eng.set_regularizer(otdr.QuadraticReg(200.0))
        eng.set_state()
        assert eng.solve_path() == ("stream" if mode == "on" else "graph")
        out[mode] = eng.solve(otdr.SolverOptions(tol_primal=1e-4, max_iter=3000, storage="f32"),
                              with_state=False)
        eng.close()
    a, b = out["on"], out["off"]
    assert a.termination.name == b.termination.name == "Converged"
    assert abs(a.iterations - b.iterations) <= 2, (a.iterations, b.iterations)
    assert abs(a.objective - b.objective) <= 1e-6 * abs(b.objective)


def test_cfg3_size_group_lasso_properties():
    """cfg3 at full size (10000^2, 10 class groups, lambda 1e-3, fp32) through
    the pipelined GL kernel: non-negativity, mass balance sum r = sum s, row
    and column sums consistent with r and s, and every (column, class) group
    either annihilated or strictly positive-normed after 25 iterations."""
    from paper_2305_18483_b200 import datagen

    m = n = 10000
    src, tgt, ls, lt = datagen.adaptation_points(m, n, 10, 0)
    p, q = datagen.uniform(m), datagen.uniform(n)
    eng = otdr.Engine(m, n, "f32")
    eng.build_sqdist_cost(src, tgt, p, q)
    eng.set_regularizer(otdr.GroupLassoReg(1e-3, otdr.column_class_blocks(ls, n)))
    eng.set_state()
    eng.step(otdr.default_stepsize(m, n), 25)
    g = eng.get_state()
    eng.close()
    assert g.k == 25
    assert (g.X >= 0).all()
    assert abs(g.r.sum() - g.s.sum()) <= 1e-9
    np.testing.assert_allclose(g.X.sum(axis=1) - p, g.r, atol=1e-9)
    np.testing.assert_allclose(g.X.sum(axis=0) - q, g.s, atol=1e-9)
    lab = np.asarray(ls)
    for c in range(10):
        norms = np.sqrt((g.X[lab == c].astype(np.float64) ** 2).sum(axis=0))
        assert np.isfinite(norms).all() and (norms >= 0).all()


@pytest.mark.parametrize("kind,param", [("none", 0.0), ("quad", 0.7), ("quad", 123.0), ("gl", 0.02)])
@pytest.mark.parametrize("resident", ["on", "off"])
def test_first_step_bitwise(ora, monkeypatch, kind, param, resident):
    """fp64 storage: the first DR step from default_init is purely element-wise
    (phi0, psi0 are constants, the sums of X0 = 0 are exact), so X_1 must equal
    the reference arithmetic BIT FOR BIT -- including the quadratic prox's true
    division (regularizers.cpp:54) and the group-lasso scale."""
    monkeypatch.setenv("OTDR_RESIDENT", resident)
    m, n = 1500, 1300
    C, p, q, *_ = ora.gaussian_problem(m, n, 41)
    labels = [i % 3 for i in range(m)]
    pr = ora.Problem(C, p, q)
    st = ora.make_state(pr)
    ora.step(st, pr, oracle_reg(ora, kind, param, labels, n), ora.default_stepsize(m, n))
    eng = otdr.Engine(m, n, "f64")
    eng.set_problem(C, p, q)
    eng.set_regularizer(dev_reg(kind, param, labels, n))
    eng.set_state()
    eng.step(ora.default_stepsize(m, n), 1)
    g = eng.get_state()
    eng.close()
    if kind == "gl":  # group norms are sums: their order differs, so 1 ulp is allowed
        assert rel(g.X, st.X) <= 1e-15
    else:
        assert np.array_equal(g.X, st.X), int((g.X != st.X).sum())


@pytest.mark.timeout(240, method="thread")  # a hung exchange must not hang the suite
def test_peer_exchange_device_cost_builder(ora, monkeypatch):
    """Row-sharded device cost builder without NCCL: the normalising maximum
    of squared_distance_cost (problem.cpp:68-74) is all-reduced (max) over
    the peer buffers, so every rank's band equals the unsharded cost."""
    monkeypatch.setenv("OTDR_STREAM_GRID", "100")
    from paper_2305_18483_b200 import datagen, sharding

    m, n = 700, 650
    src, tgt = datagen.gaussian_points(m, n, 9)
    p, q = datagen.uniform(m), datagen.uniform(n)
    full = otdr.Engine(m, n, "f64")
    full.build_sqdist_cost(src, tgt, p, q)
    full.set_regularizer(otdr.QuadraticReg(1.0))
    full.set_state()
    full.step(otdr.default_stepsize(m, n), 6)
    ref = full.get_state()
    full.close()
    bands = sharding.row_bands(m, 2)
    engs = [otdr.Engine(m, n, "f64", shard=otdr.Shard(r, 2, lo, hi, None)) for r, (lo, hi) in enumerate(bands)]
    otdr.link_local(engs)
    _parallel([lambda e=e, lo=lo, hi=hi: e.build_sqdist_cost(src[lo:hi], tgt, p[lo:hi], q)
               for e, (lo, hi) in zip(engs, bands)])
    for e in engs:
        e.set_regularizer(otdr.QuadraticReg(1.0))
    _parallel([e.set_state for e in engs])
    _parallel([lambda e=e: e.step(otdr.default_stepsize(m, n), 6) for e in engs])
    gs = _parallel([e.get_state for e in engs])
    X = np.concatenate([g.X for g in gs])
    assert rel(X, ref.X) <= 1e-12, rel(X, ref.X)
    for e in engs:
        e.close()


@pytest.mark.parametrize("storage", ["f64", "f32"])
@pytest.mark.parametrize("m,n,classes", [(1200, 900, 4), (3000, 700, 3), (1000, 1000, 10)])
def test_gl_stream_kernel_matches_oracle_and_graph(ora, monkeypatch, storage, m, n, classes):
    """Persistent group-lasso solve (gl_stream_kernel, one launch) against the
    oracle after k steps, and a full solve against the graph loop
    (OTDR_GL_STREAM=off): same termination and iteration count."""
    C, p, q, src, tgt, ls, lt = ora.adaptation_problem(m, n, classes, 13)
    Co = C if storage == "f64" else C.astype(np.float32).astype(np.float64)
    pr = ora.Problem(Co, p, q)
    offs, cells = ora.column_class_blocks(ls, n)
    oreg = ora.group_lasso_reg(2e-3, offs, cells)
    st = ora.make_state(pr)
    reg = otdr.GroupLassoReg(2e-3, otdr.column_class_blocks(ls, n))
    eng = otdr.Engine(m, n, storage)
    eng.set_problem(C, p, q)
    eng.set_regularizer(reg)
    eng.set_state()
    assert eng.solve_path() == "stream"
    rho = ora.default_stepsize(m, n)
    tol = 1e-12 if storage == "f64" else 1e-5
    done = 0
    for k in (1, 8, 30):
        for _ in range(k - done):
            ora.step(st, pr, oreg, rho)
        eng.step(rho, k - done)
        done = k
        g = eng.get_state()
        assert g.k == k
        assert rel(g.X, st.X) <= tol, (k, rel(g.X, st.X))
        assert rel(g.phi, st.phi) <= tol and rel(g.psi, st.psi) <= tol
    eng.set_state()
    a = eng.solve(otdr.SolverOptions(tol_primal=1e-5, max_iter=5000, storage=storage), with_state=False)
    eng.close()
    monkeypatch.setenv("OTDR_GL_STREAM", "off")
    eng = otdr.Engine(m, n, storage)
    eng.set_problem(C, p, q)
    eng.set_regularizer(reg)
    eng.set_state()
    assert eng.solve_path() == "graph"
    b = eng.solve(otdr.SolverOptions(tol_primal=1e-5, max_iter=5000, storage=storage), with_state=False)
    eng.close()
    assert a.termination == b.termination
    assert abs(a.iterations - b.iterations) <= (0 if storage == "f64" else 2)
    assert abs(a.objective - b.objective) <= (1e-9 if storage == "f64" else 1e-6) * abs(b.objective)


@pytest.mark.parametrize("path", ["resident", "stream", "gl_stream", "graph"])
def test_nonfinite_every_device_loop(ora, monkeypatch, path):
    """solver.cpp:181-185 through every device loop: a warm start that
    overflows on the first step raises NonFiniteIterate with the reference's
    message at iteration 1 (the persistent kernels stop inside the launch)."""
    if path != "resident":
        monkeypatch.setenv("OTDR_RESIDENT", "off")
    if path == "graph":
        monkeypatch.setenv("OTDR_STREAM", "off")
        monkeypatch.setenv("OTDR_GL_STREAM", "off")
    m, n = 300, 280
    C, p, q, *_ = ora.gaussian_problem(m, n, 3)
    pr = otdr.validate_problem(C, p, q)
    reg = (otdr.GroupLassoReg(1e-3, otdr.column_class_blocks([i % 3 for i in range(m)], n))
           if path == "gl_stream" else otdr.ZeroReg())
    init = otdr.WarmStart(np.full((m, n), 1e308), np.zeros(m), np.zeros(n))
    with pytest.raises(otdr.NonFiniteIterate, match="non-finite iterate at iteration 1"):
        otdr.solve(pr, reg, otdr.SolverOptions(init=init, storage="f64"))


@pytest.mark.parametrize("max_iter", [40, 41])  # ends after an odd / an even (shifted) iteration
@pytest.mark.parametrize("kind,param", [("none", 0.0), ("quad", 0.9)])
def test_fused_stream_kernel_matches_oracle(ora, monkeypatch, kind, param, max_iter):
    """SolverOptions.fused (solver.cpp:127-177) on the streaming kernel, fp64:
    even iterations store B = X - rho C, odd ones read B and never C. Same
    iterations, plan (un-shifted when the run ends on an even step), phi and
    objective as the oracle's fused solve."""
    monkeypatch.setenv("OTDR_RESIDENT", "off")
    m, n = 700, 600
    C, p, q, *_ = ora.gaussian_problem(m, n, 23)
    pr = ora.Problem(C, p, q)
    o = ora.solve(pr, oracle_reg(ora, kind, param, None, n), max_iter=max_iter, tol_primal=1e-300,
                  fused=True)
    eng = otdr.Engine(m, n, "f64")
    eng.set_problem(C, p, q)
    eng.set_regularizer(dev_reg(kind, param, None, n))
    eng.set_state()
    assert eng.solve_path() == "stream"
    rep = eng.solve(otdr.SolverOptions(max_iter=max_iter, tol_primal=1e-300, fused=True, storage="f64"))
    eng.close()
    assert rep.iterations == o.iterations == max_iter
    assert rel(rep.plan(), o.state.X) <= 1e-12, rel(rep.plan(), o.state.X)
    assert rel(rep.state.phi, o.state.phi) <= 1e-12 and rel(rep.state.psi, o.state.psi) <= 1e-12
    assert abs(rep.objective - o.objective) <= 1e-11 * abs(o.objective)


@pytest.mark.parametrize("kind,param,tol_gap", [("quad", 0.5, 1e-7), ("none", 0.0, 1e-6), ("gl", 1e-3, 1e-6)])
def test_tol_gap_on_persistent_kernels(ora, monkeypatch, kind, param, tol_gap):
    """tol_gap (solver.cpp:205-219) on the persistent kernels: a launch stops at
    every check iteration with r_primal <= tol, the certificate kernels decide
    (Converged / continue / Stalled / MaxIter), the host relaunches. Same
    termination, iteration count and final objective as the oracle."""
    monkeypatch.setenv("OTDR_RESIDENT", "off")
    m, n = 400, 350
    C, p, q, *_ = ora.gaussian_problem(m, n, 29)
    labels = [i % 4 for i in range(m)]
    pr = ora.Problem(C, p, q)
    o = ora.solve(pr, oracle_reg(ora, kind, param, labels, n), tol_primal=1e-6, tol_gap=tol_gap,
                  check_every=5, max_iter=30000)
    eng = otdr.Engine(m, n, "f64")
    eng.set_problem(C, p, q)
    eng.set_regularizer(dev_reg(kind, param, labels, n))
    eng.set_state()
    assert eng.solve_path() == "stream"
    rep = eng.solve(otdr.SolverOptions(tol_primal=1e-6, tol_gap=tol_gap, check_every=5, max_iter=30000,
                                       storage="f64"))
    eng.close()
    assert rep.termination.name == o.termination
    assert rep.iterations == o.iterations
    assert abs(rep.objective - o.objective) <= 1e-10 * abs(o.objective)


@pytest.mark.parametrize("kernel", ["tma", "async"])
@pytest.mark.parametrize("m,n", [(3, 4000), (5, 3000), (33, 257), (300, 517), (1500, 1400), (2100, 2501)])
@pytest.mark.parametrize("kind,param", [("none", 0.0), ("quad", 0.7)])
def test_fp32_stream_kernels_match_oracle(ora, monkeypatch, kernel, m, n, kind, param):
    """fp32 storage through both persistent streaming kernels -- the TMA
    producer-warp kernel (tstream_kernel, the default: 8-row blocks, so m < 8
    and tiles ending mid-block are covered) and the per-thread cp.async kernel
    -- against the oracle on the fp32-rounded cost: iterates after k steps
    within 1e-5, then a full solve (same termination, iterations within 2,
    objective within 1e-6)."""
    monkeypatch.setenv("OTDR_RESIDENT", "off")
    monkeypatch.setenv("OTDR_STREAM_KERNEL", kernel)
    C, p, q, *_ = ora.gaussian_problem(m, n, 23 + m)
    pr = ora.Problem(C.astype(np.float32).astype(np.float64), p, q)
    alpha = param * (m + n)
    oreg = oracle_reg(ora, kind, alpha, None, n)
    st = ora.make_state(pr)
    eng = otdr.Engine(m, n, "f32")
    eng.set_problem(C, p, q)
    eng.set_regularizer(dev_reg(kind, alpha, None, n))
    eng.set_state()
    assert eng.solve_path() == "stream"
    assert eng.kernel_name().startswith("tstream_kernel" if kernel == "tma" else "stream_kernel")
    rho = ora.default_stepsize(m, n)
    done = 0
    for k in (1, 9, 60):
        for _ in range(k - done):
            ora.step(st, pr, oreg, rho)
        eng.step(rho, k - done)
        done = k
        g = eng.get_state()
        assert g.k == st.k == k
        for nm in ("X", "phi", "psi", "a", "b"):
            assert rel(getattr(g, nm), getattr(st, nm)) <= 1e-5, (k, nm)
    o = ora.solve(pr, oreg, tol_primal=1e-6, max_iter=5000)
    eng.set_state()
    rep = eng.solve(otdr.SolverOptions(tol_primal=1e-6, max_iter=5000, storage="f32"), with_state=False)
    assert rep.termination.name == o.termination
    assert abs(rep.iterations - o.iterations) <= 2
    assert abs(rep.objective - o.objective) <= 1e-6 * max(abs(o.objective), 1e-300)
    eng.close()


@pytest.mark.parametrize("ts_cfg", ["1", "2"])
@pytest.mark.parametrize("m,n", [(5, 3000), (300, 517), (2100, 2501)])
def test_tstream_geometries_match_oracle(ora, monkeypatch, ts_cfg, m, n):
    """The non-default TMA-kernel geometries (OTDR_TS_CFG=1: 8 consumer warps
    x 1 row, 5 stages, 2 CTAs/SM; 2: 16 warps, 16-row blocks) against the
    oracle on the fp32-rounded cost, like the default geometry in
    test_fp32_stream_kernels_match_oracle: iterates after k steps within 1e-5,
    a full solve to the same termination, iterations within 2."""
    monkeypatch.setenv("OTDR_RESIDENT", "off")
    monkeypatch.setenv("OTDR_TS_CFG", ts_cfg)
    C, p, q, *_ = ora.gaussian_problem(m, n, 41 + m)
    pr = ora.Problem(C.astype(np.float32).astype(np.float64), p, q)
    alpha = 0.7 * (m + n)
    oreg = oracle_reg(ora, "quad", alpha, None, n)
    st = ora.make_state(pr)
    eng = otdr.Engine(m, n, "f32")
    eng.set_problem(C, p, q)
    eng.set_regularizer(dev_reg("quad", alpha, None, n))
    eng.set_state()
    assert eng.solve_path() == "stream"
    assert eng.kernel_name().startswith("tstream_kernel")
    rho = ora.default_stepsize(m, n)
    done = 0
    for k in (1, 20):
        for _ in range(k - done):
            ora.step(st, pr, oreg, rho)
        eng.step(rho, k - done)
        done = k
        g = eng.get_state()
        for nm in ("X", "phi", "psi", "a", "b"):
            assert rel(getattr(g, nm), getattr(st, nm)) <= 1e-5, (k, nm)
    o = ora.solve(pr, oreg, tol_primal=1e-6, max_iter=5000)
    eng.set_state()
    rep = eng.solve(otdr.SolverOptions(tol_primal=1e-6, max_iter=5000, storage="f32"), with_state=False)
    assert rep.termination.name == o.termination
    assert abs(rep.iterations - o.iterations) <= 2
    assert abs(rep.objective - o.objective) <= 1e-6 * max(abs(o.objective), 1e-300)
    eng.close()


@pytest.mark.parametrize("m,n,kind", [(20, 20, "none"), (300, 517, "quad"), (1000, 1000, "quad")])
def test_resident_f32_storage_runs_fp64_tiles(ora, m, n, kind):
    """fp32 storage on the resident loop: the iteration runs on fp64 tiles of
    the fp32-rounded cost, so after k steps in one launch the state equals the
    oracle's fp64 DR on that cost up to the final fp32 rounding of X (and
    phi / psi to fp64 reduction order)."""
    C, p, q, *_ = ora.gaussian_problem(m, n, 2)
    pr = ora.Problem(C.astype(np.float32).astype(np.float64), p, q)
    alpha = 5e-3 * (m + n)
    oreg = oracle_reg(ora, kind, alpha, None, n)
    st = ora.make_state(pr)
    eng = otdr.Engine(m, n, "f32")
    eng.set_problem(C, p, q)
    eng.set_regularizer(dev_reg(kind, alpha, None, n))
    eng.set_state()
    assert eng.solve_path() == "resident"
    assert "f64 tiles" in eng.kernel_name()
    rho = ora.default_stepsize(m, n)
    for _ in range(37):
        ora.step(st, pr, oreg, rho)
    eng.step(rho, 37)
    g = eng.get_state()
    eng.close()
    assert rel(g.X, st.X) <= 1e-7
    for nm in ("phi", "psi", "a", "b"):
        assert rel(getattr(g, nm), getattr(st, nm)) <= 1e-10, nm
