"""Committed golden fixtures (tests/golden/*.npz, made by tests/golden/make_golden.py).

CPU: the pinned oracle still reproduces every fixture bit for bit (guards the
checker against drift). GPU: the sm_100a path, through the C-ABI, against the
stored vectors -- K raw steps (fp64 storage <= 1e-12 relative, fp32 storage
<= 1e-5 relative: the north star's iterate tolerance) and solve() (same
iteration count and termination, objective within 1e-6).
"""
import glob
import os

import numpy as np
import pytest

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FILES = sorted(glob.glob(os.path.join(HERE, "*.npz")))
NAMES = [os.path.basename(f)[:-4] for f in FILES]


def load(name):
    with np.load(os.path.join(HERE, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def test_fixtures_present():
    assert set(NAMES) >= {"quad_48x40", "zero_33x57", "gl_60x50", "gl_random_20x20"}


@pytest.mark.parametrize("name", NAMES)
def test_oracle_reproduces_golden(ora, name):
    import importlib.util

    spec = importlib.util.spec_from_file_location("make_golden", os.path.join(HERE, "make_golden.py"))
    mg = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mg)
    g = load(name)
    d = mg.make(name)
    for key, v in g.items():
        assert np.array_equal(np.asarray(d[key]), v), (name, key)


def _dev_reg(otdr, g):
    kind, param, n = str(g["kind"]), float(g["param"]), g["C"].shape[1]
    if kind == "none":
        return otdr.ZeroReg()
    if kind == "quad":
        return otdr.QuadraticReg(param)
    return otdr.GroupLassoReg(param, otdr.column_class_blocks([int(v) for v in g["labels"]], n))


@pytest.mark.gpu
@pytest.mark.parametrize("storage,tol", [("f64", 1e-12), ("f32", 1e-5)])
@pytest.mark.parametrize("name", NAMES)
def test_device_steps_match_golden(name, storage, tol):
    otdr = pytest.importorskip("paper_2305_18483_b200")
    g = load(name)
    m, n = g["C"].shape
    eng = otdr.Engine(m, n, storage)
    try:
        eng.set_problem(g["C"], g["p"], g["q"])
        eng.set_regularizer(_dev_reg(otdr, g))
        eng.set_state()
        eng.step(float(g["rho"]), int(g["k"]))
        st = eng.get_state()
    finally:
        eng.close()
    assert st.k == int(g["k"])
    for key in ("X", "phi", "psi", "a", "b"):
        assert rel(getattr(st, key), g[key]) <= tol, (key, rel(getattr(st, key), g[key]))
    assert abs(st.theta - float(g["theta"])) <= tol * max(1.0, abs(float(g["theta"])))


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_device_solve_matches_golden(name):
    otdr = pytest.importorskip("paper_2305_18483_b200")
    g = load(name)
    opts = otdr.SolverOptions(tol_primal=float(g["solve_tol"]), max_iter=200000)
    rep = otdr.solve(otdr.Problem(g["C"], g["p"], g["q"]), _dev_reg(otdr, g), opts)
    assert rep.termination.name == str(g["solve_termination"])
    assert rep.iterations == int(g["solve_iterations"])
    obj = float(g["solve_objective"])
    assert abs(rep.objective - obj) <= 1e-6 * max(1.0, abs(obj))
    assert rel(rep.plan(), g["solve_X"]) <= 1e-9
