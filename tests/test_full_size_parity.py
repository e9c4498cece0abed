"""Full-size parity: the device path against the CPU oracle at the sizes the
numbers in bench.py / DESIGN.md are quoted on (BASELINE.json configs).

Two kinds of evidence:

  * live k-step iterates -- the oracle (oracle/otdr_oracle.cpp, all host
    threads) and the device both run k in {1, 10, 100} raw DR steps
    (solver.cpp:95-102 + :23-38) from make_state on the same seeded instance
    (datagen.cpp:56-65 / :67-129); X (every entry), phi, psi, a, b within 1e-5
    relative (max-norm) for fp32 storage, 1e-12 for fp64 storage. The oracle
    runs on the fp32-rounded cost for fp32 storage (what the device holds).
  * complete solves to r_primal <= 1e-4 against goldens the oracle produced
    once (tests/golden/make_full_size.py; a 20000^2 oracle solve takes
    minutes): same termination; stopping iteration K within the stated
    tolerance (fp64 storage: identical); objective within 1e-6 relative of
    the oracle's objective AT THE DEVICE'S stopping iteration; r_primal
    within 1e-6 absolute of the oracle's at that iteration; and the state
    after exactly K raw steps (phi, psi, a, b, r, s, six plan rows, sum X,
    sum X^2) within 1e-5 relative (fp64: 1e-10).

A CPU test (not gpu) checks that the oracle still reproduces the first goldens'
r_primal values bit for bit (drift guard).
"""
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "full")
THREADS = os.cpu_count() or 1


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def rel_rows(a, b, chunk=2000):
    """rel() without full-size temporaries (40000^2 plans)."""
    num, den = 0.0, 0.0
    for i in range(0, a.shape[0], chunk):
        num = max(num, float(np.abs(a[i:i + chunk] - b[i:i + chunk]).max()))
        den = max(den, float(np.abs(b[i:i + chunk]).max()))
    return num / max(den, 1e-300)


def golden(name):
    path = os.path.join(GOLD, f"full_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (tests/golden/make_full_size.py)")
    return np.load(path)


# ------------------------------------------------------------------ CPU drift guard
def test_cfg2_golden_trace_reproduced_by_oracle(ora):
    """The oracle's first 3 r_primal values at cfg2 (10000^2, zero reg, fp32
    cost) equal the committed golden's bit for bit."""
    g = golden("cfg2_f32")
    C, p, q, *_ = ora.gaussian_problem(10000, 10000, 0)
    C = C.astype(np.float32).astype(np.float64)
    pr = ora.Problem(C, p, q)
    st = ora.make_state(pr)
    rho = ora.default_stepsize(10000, 10000)
    assert rho == float(g["rho"])
    for k in range(3):
        ora.step(st, pr, ora.zero_reg(), rho, THREADS)
        nr, ns = float(np.sqrt(np.dot(st.r, st.r))), float(np.sqrt(np.dot(st.s, st.s)))
        assert (ns if nr < ns else nr) == float(g["r_primal_trace"][k])


def test_full_size_goldens_consistent():
    """Each golden stops at its first iteration with r_primal <= tol."""
    for name in ("headline_f32", "headline_f64", "cfg2_f32", "cfg3_f32"):
        g = golden(name)
        K, tr, tol = int(g["iterations"]), g["r_primal_trace"], float(g["tol"])
        assert tr[K - 1] <= tol and (tr[: K - 1] > tol).all()
        assert K in set(int(v) for v in g["obj_iter"])
    c5 = golden("cfg5_f32")
    assert c5["iterations"].shape == (256,) and (c5["r_primal"] <= 1e-4).all()


# ------------------------------------------------------------------ GPU
gpu = pytest.mark.gpu


def _otdr():
    return pytest.importorskip("paper_2305_18483_b200")


def _gaussian_engine(otdr, m, n, seed, storage):
    from paper_2305_18483_b200 import datagen

    eng = otdr.Engine(m, n, storage)
    src, tgt = datagen.gaussian_points(m, n, seed)
    eng.build_sqdist_cost(src, tgt, datagen.uniform(m), datagen.uniform(n))
    return eng


def _adaptation_engine(otdr, m, n, classes, seed, storage):
    from paper_2305_18483_b200 import datagen

    eng = otdr.Engine(m, n, storage)
    src, tgt, ls, lt = datagen.adaptation_points(m, n, classes, seed)
    eng.build_sqdist_cost(src, tgt, datagen.uniform(m), datagen.uniform(n))
    return eng, ls


def _dev_reg(otdr, kind, param, labels, n):
    if kind == "none":
        return otdr.ZeroReg()
    if kind == "quad":
        return otdr.QuadraticReg(param)
    return otdr.GroupLassoReg(param, otdr.column_class_blocks(labels, n))


def _ora_reg(ora, kind, param, labels, n):
    if kind == "none":
        return ora.zero_reg()
    if kind == "quad":
        return ora.quad_reg(param)
    return ora.group_lasso_reg(param, *ora.column_class_blocks(labels, n))


def _live_k_steps(ora, otdr, case, storage, ks=(1, 10, 100)):
    """Oracle and device run the same raw steps; compare after each k in ks."""
    kind, param, m, n = case["kind"], case["param"], case["m"], case["n"]
    if case["gen"] == "gaussian":
        C, p, q, *_ = ora.gaussian_problem(m, n, 0)
        labels = None
        eng = _gaussian_engine(otdr, m, n, 0, storage)
    else:
        C, p, q, _, _, labels, _ = ora.adaptation_problem(m, n, case["classes"], 0)
        eng, _ = _adaptation_engine(otdr, m, n, case["classes"], 0, storage)
    if storage == "f32":
        C32 = C.astype(np.float32)
        C[...] = C32
        del C32
    pr = ora.Problem(C, p, q)
    oreg = _ora_reg(ora, kind, param, labels, n)
    st = ora.make_state(pr)
    eng.set_regularizer(_dev_reg(otdr, kind, param, labels, n))
    eng.set_state()
    rho = ora.default_stepsize(m, n)
    tol = 1e-5 if storage == "f32" else 1e-12
    plan = np.empty((m, n))
    done = 0
    out = {}
    for k in ks:
        for _ in range(k - done):
            ora.step(st, pr, oreg, rho, THREADS)
        eng.step(rho, k - done)
        done = k
        g = eng.get_state(with_plan=False)
        eng.get_plan_into(plan)
        assert g.k == st.k == k
        errs = {"X": rel_rows(plan, st.X), "phi": rel(g.phi, st.phi), "psi": rel(g.psi, st.psi),
                "a": rel(g.a, st.a), "b": rel(g.b, st.b)}
        out[k] = errs
        for nm, e in errs.items():
            assert e <= tol, (k, nm, e)
        assert abs(g.theta - st.theta) <= tol * max(1.0, abs(st.theta))
    eng.close()
    print(f"live k-steps {case} {storage}: {out}")
    return out


HEADLINE = dict(gen="gaussian", kind="quad", param=200.0, m=20000, n=20000)
CFG2 = dict(gen="gaussian", kind="none", param=0.0, m=10000, n=10000)
CFG3 = dict(gen="adaptation", classes=10, kind="gl", param=1e-3, m=10000, n=10000)
CFG4 = dict(gen="gaussian", kind="quad", param=400.0, m=40000, n=40000)


@gpu
@pytest.mark.timeout(1200, method="thread")
@pytest.mark.parametrize("storage", ["f32", "f64"])
def test_headline_k_steps_vs_oracle(ora, storage):
    """20000^2 quadratic alpha = 200 (the bench config): k in {1, 10, 100}."""
    _live_k_steps(ora, _otdr(), HEADLINE, storage)


@gpu
@pytest.mark.timeout(1200, method="thread")
def test_cfg2_k_steps_vs_oracle(ora):
    """cfg2: unregularized 10000^2 fp32 on the reference generator."""
    _live_k_steps(ora, _otdr(), CFG2, "f32")


@gpu
@pytest.mark.timeout(1200, method="thread")
def test_cfg3_k_steps_vs_oracle(ora):
    """cfg3: group lasso 10000^2, 10 class row groups, lambda 1e-3, fp32."""
    _live_k_steps(ora, _otdr(), CFG3, "f32")


@gpu
@pytest.mark.timeout(1800, method="thread")
def test_cfg4_k_steps_vs_oracle(ora):
    """cfg4: quadratic 40000^2 (alpha = 400) on one GPU, k in {1, 10}."""
    try:
        import psutil

        if psutil.virtual_memory().available < 72e9:
            pytest.skip("cfg4 oracle needs ~60 GB of host memory")
    except ImportError:
        pass
    _live_k_steps(ora, _otdr(), CFG4, "f32", ks=(1, 10))


@gpu
@pytest.mark.timeout(1200, method="thread")
def test_headline_fused_vs_oracle_fused(ora):
    """solve(fused=True) at 20000^2 fp32 (max_iter 100) against the oracle's
    fused even/odd solve (solver.cpp:127-177) on the same inputs."""
    otdr = _otdr()
    m = n = 20000
    C, p, q, *_ = ora.gaussian_problem(m, n, 0)
    C[...] = C.astype(np.float32)
    o = ora.solve(ora.Problem(C, p, q), ora.quad_reg(200.0), tol_primal=1e-300, max_iter=100,
                  fused=True, threads=THREADS)
    del C
    eng = _gaussian_engine(otdr, m, n, 0, "f32")
    eng.set_regularizer(otdr.QuadraticReg(200.0))
    eng.set_state()
    rep = eng.solve(otdr.SolverOptions(tol_primal=1e-300, max_iter=100, storage="f32", fused=True),
                    with_state=True)
    eng.close()
    g = rep.state
    assert rep.iterations == o.iterations == 100 and rep.termination.name == o.termination
    for nm in ("X", "phi", "psi", "a", "b"):
        e = rel_rows(getattr(g, nm), getattr(o.state, nm)) if nm == "X" else \
            rel(getattr(g, nm), getattr(o.state, nm))
        assert e <= 1e-5, (nm, e)
    assert abs(rep.objective - o.objective) <= 1e-6 * abs(o.objective)


def _solve_vs_golden(otdr, name, make_engine, storage, fused=False, k_tol=2):
    g = golden(name)
    m, n, K = int(g["m"]), int(g["n"]), int(g["iterations"])
    tol = float(g["tol"])
    eng = make_engine()
    eng.set_state()
    rep = eng.solve(otdr.SolverOptions(tol_primal=tol, max_iter=3 * K, storage=storage, fused=fused),
                    with_state=False)
    assert rep.termination.name == str(g["termination"]) == "Converged"
    Kd = rep.iterations
    assert abs(Kd - K) <= k_tol, (Kd, K)
    tr = g["r_primal_trace"]
    assert abs(rep.r_primal - tr[Kd - 1]) <= 1e-6, (rep.r_primal, tr[Kd - 1])
    oi = list(int(v) for v in g["obj_iter"])
    assert Kd in oi, (Kd, oi)
    obj = float(g["obj_val"][oi.index(Kd)])
    assert abs(rep.objective - obj) <= 1e-6 * abs(obj), (rep.objective, obj)
    # the state after exactly the oracle's K raw steps
    eng.set_state()
    eng.step(float(g["rho"]), K)
    st = eng.get_state(with_plan=False)
    plan = np.empty((m, n))
    eng.get_plan_into(plan)
    eng.close()
    vt = 1e-5 if storage == "f32" else 1e-10
    errs = {nm: rel(getattr(st, nm), g[nm]) for nm in ("phi", "psi", "a", "b", "r", "s")}
    errs["plan_rows"] = rel(plan[g["rows"]], g["plan_rows"])
    errs["x_sum"] = abs(float(plan.sum()) - float(g["x_sum"])) / abs(float(g["x_sum"]))
    errs["x_sumsq"] = abs(float(np.einsum("ij,ij->", plan, plan)) - float(g["x_sumsq"])) / float(g["x_sumsq"])
    print(f"{name} {storage}{' fused' if fused else ''}: K device {Kd} oracle {K}; "
          f"objective {rep.objective!r} vs {obj!r}; state errs {errs}")
    for nm, e in errs.items():
        assert e <= vt, (nm, e)
    assert abs(st.theta - float(g["theta"])) <= vt * max(1.0, abs(float(g["theta"])))


@gpu
@pytest.mark.timeout(1200, method="thread")
@pytest.mark.parametrize("storage,fused", [("f32", False), ("f32", True), ("f64", False)])
def test_headline_solve_vs_golden(storage, fused):
    """The bench config solved to 1e-4: fp32 (plain and fused=True) vs the
    oracle on the fp32 cost, fp64 vs the oracle on the fp64 cost (K exact)."""
    otdr = _otdr()

    def mk():
        eng = _gaussian_engine(otdr, 20000, 20000, 0, storage)
        eng.set_regularizer(otdr.QuadraticReg(200.0))
        return eng

    _solve_vs_golden(otdr, f"headline_{storage}", mk, storage, fused=fused,
                     k_tol=0 if storage == "f64" else 2)


@gpu
@pytest.mark.timeout(1200, method="thread")
def test_cfg2_solve_vs_golden():
    otdr = _otdr()

    def mk():
        eng = _gaussian_engine(otdr, 10000, 10000, 0, "f32")
        eng.set_regularizer(otdr.ZeroReg())
        return eng

    _solve_vs_golden(otdr, "cfg2_f32", mk, "f32")


@gpu
@pytest.mark.timeout(1200, method="thread")
def test_cfg3_solve_vs_golden():
    otdr = _otdr()

    def mk():
        eng, ls = _adaptation_engine(otdr, 10000, 10000, 10, 0, "f32")
        eng.set_regularizer(otdr.GroupLassoReg(1e-3, otdr.column_class_blocks(ls, 10000)))
        return eng

    _solve_vs_golden(otdr, "cfg3_f32", mk, "f32")


@gpu
@pytest.mark.timeout(1200, method="thread")
def test_cfg5_batch_256_vs_golden():
    """cfg5: 256 x 512^2 quadratic (alpha 5.12), fp32, one batched launch vs
    256 oracle solve()s: per-problem termination, iterations (+-3: fp32
    storage vs fp64 arithmetic near the threshold), objective (1e-6) and
    r_primal (<= tol, within 1e-6 of the oracle's)."""
    otdr = _otdr()
    from paper_2305_18483_b200 import datagen

    g = golden("cfg5_f32")
    B, m = int(g["B"]), int(g["m"])
    src = np.empty((B, m, 2))
    tgt = np.empty((B, m, 2))
    for b in range(B):
        src[b], tgt[b] = datagen.gaussian_points(m, m, b)
    ps = np.full((B, m), 1.0 / m)
    be = otdr.BatchEngine(B, m, m, "f32")
    be.build_sqdist_costs(src, tgt, ps, ps)
    be.set_regularizer(otdr.QuadraticReg(float(g["alpha"])))
    reps = be.solve(otdr.SolverOptions(tol_primal=float(g["tol"]), max_iter=20000))
    sts = be.states(with_plan=False)
    be.close()
    it = np.array([r.iterations for r in reps])
    dk = np.abs(it - g["iterations"])
    print(f"cfg5: iterations device {it.sum()} oracle {int(g['iterations'].sum())}, "
          f"max |dK| {dk.max()}, exact {(dk == 0).sum()}/{B}")
    assert all(r.termination.name == "Converged" for r in reps)
    assert dk.max() <= 3
    for b, r in enumerate(reps):
        assert abs(r.objective - g["objective"][b]) <= 1e-6 * abs(g["objective"][b]), b
        assert r.r_primal <= float(g["tol"])
        assert sts[b].k == r.iterations
        if dk[b] == 0:
            assert abs(r.r_primal - g["r_primal"][b]) <= 1e-6
