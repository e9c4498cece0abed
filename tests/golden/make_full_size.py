#!/usr/bin/env python
"""Full-size oracle goldens for the BASELINE.json configurations (test data, not product code).

The GPU numbers in bench.py / DESIGN.md are quoted on full-size instances whose
complete solves take the CPU oracle minutes (20000^2: ~1150 iterations at
~0.15-0.5 s each). Those solves are run ONCE here and their results frozen
under tests/golden/full/full_*.npz; tests/test_full_size_parity.py then checks the
device path against them on the GPU box (where /root/reference does not exist
and the oracle is too slow to re-run a full solve per test run). The k-step
iterate checks at full size run the oracle live instead (tests/test_full_size_parity.py).

Oracle: oracle/otdr_oracle.cpp (pinned to the reference's KATs in
tests/test_oracle_kats.py), following /root/reference/proj/src/solver.cpp:95-102
(step), :23-38 (recurrence), :104-241 (solve: r_primal = max(|r|, |s|) at
:179, converged when r_primal <= tol at a check iteration :218, iterations =
st.k), problem.cpp:76-85 (primal_objective), on inputs from datagen.cpp:56-65 /
:67-129 (restated bit-exactly).

fp32-storage cases run the oracle on the fp32-rounded cost (C32 = float(C)),
which is exactly what the device holds; the oracle's arithmetic stays fp64.

Each case stores:
  * iterations K, termination, r_primal trace (every iteration 1..K+4)
  * objective at every iteration from the first with r_primal <= 1.25 tol
    through K+4 (so a device run stopping a few iterations away from K is
    compared at its own stopping iteration)
  * the state at K: phi, psi, a, b, r, s, theta, eta, selected plan rows,
    sum(X), sum(X^2), nnz(X)

  python tests/golden/make_full_size.py [case ...]    # rewrites tests/golden/full/full_<case>.npz
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import pyoracle as ora  # noqa: E402

THREADS = os.cpu_count() or 1
EXTRA = 4  # iterations recorded past K


def gaussian(m, n, seed, f32):
    C, p, q, *_ = ora.gaussian_problem(m, n, seed)
    if f32:
        C = C.astype(np.float32).astype(np.float64)
    return C, p, q, None


def adaptation(m, n, classes, seed, f32):
    C, p, q, src, tgt, ls, lt = ora.adaptation_problem(m, n, classes, seed)
    if f32:
        C = C.astype(np.float32).astype(np.float64)
    return C, p, q, ls


# name: (inputs, regularizer kind, parameter, tol, max_iter, plan rows to keep)
CASES = {
    # the bench.py headline: gaussian_problem(20000,20000,0), QuadraticReg(5e-3 (m+n) = 200)
    "headline_f32": (lambda: gaussian(20000, 20000, 0, True), "quad", 200.0, 1e-4, 3000),
    "headline_f64": (lambda: gaussian(20000, 20000, 0, False), "quad", 200.0, 1e-4, 3000),
    # cfg2: unregularized DROT 10000^2 fp32 on the reference generator
    "cfg2_f32": (lambda: gaussian(10000, 10000, 0, True), "none", 0.0, 1e-4, 5000),
    # cfg3: group lasso 10000^2, 10 class row groups, lambda 1e-3
    "cfg3_f32": (lambda: adaptation(10000, 10000, 10, 0, True), "gl", 1e-3, 1e-4, 5000),
}


def oracle_reg(kind, param, labels, n):
    if kind == "none":
        return ora.zero_reg()
    if kind == "quad":
        return ora.quad_reg(param)
    offs, cells = ora.column_class_blocks(labels, n)
    return ora.group_lasso_reg(param, offs, cells)


def rprimal(st):
    # solver.cpp:179: max(|r|_2, |s|_2) (std::max: second argument when equal)
    nr, ns = float(np.sqrt(np.dot(st.r, st.r))), float(np.sqrt(np.dot(st.s, st.s)))
    return ns if nr < ns else nr


def run_case(name):
    gen, kind, param, tol, max_iter = CASES[name]
    t0 = time.time()
    C, p, q, labels = gen()
    m, n = C.shape
    pr = ora.Problem(C, p, q)
    reg = oracle_reg(kind, param, labels, n)
    rho = ora.default_stepsize(m, n)
    st = ora.make_state(pr)
    rows = np.unique(np.array([0, 1, m // 3, m // 2, (2 * m) // 3, m - 1]))
    trace, obj_iter, obj_val = [], [], []
    K = None
    snap = None
    while True:
        ora.step(st, pr, reg, rho, THREADS)
        k = st.k
        rp = rprimal(st)
        trace.append(rp)
        if not np.isfinite(rp):
            raise RuntimeError(f"{name}: non-finite iterate at {k}")
        if rp <= 1.25 * tol or (K is not None):
            obj_iter.append(k)
            obj_val.append(ora.primal_objective(pr, st.X, reg))
        if K is None and rp <= tol:
            K = k
            snap = dict(phi=st.phi.copy(), psi=st.psi.copy(), a=st.a.copy(), b=st.b.copy(),
                        r=st.r.copy(), s=st.s.copy(), theta=st.theta, eta=st.eta,
                        plan_rows=st.X[rows].copy(), x_sum=float(st.X.sum()),
                        x_sumsq=float(np.einsum("ij,ij->", st.X, st.X)),
                        x_nnz=int(np.count_nonzero(st.X)), objective=obj_val[-1],
                        r_primal=rp)
        if K is not None and k >= K + EXTRA:
            break
        if K is None and k >= max_iter:
            raise RuntimeError(f"{name}: no convergence within {max_iter}")
        if k % 100 == 0:
            print(f"  {name}: k={k} r_primal={rp:.3e} ({time.time() - t0:.0f} s)", flush=True)
    out = os.path.join(HERE, "full", f"full_{name}.npz")
    np.savez_compressed(out, m=m, n=n, kind=kind, param=param, tol=tol, rho=rho, iterations=K,
                        termination="Converged", r_primal_trace=np.array(trace),
                        obj_iter=np.array(obj_iter), obj_val=np.array(obj_val), rows=rows,
                        **snap)
    print(f"{name}: K={K} objective={snap['objective']!r} ({time.time() - t0:.0f} s) -> {out}",
          flush=True)


def run_cfg5():
    """cfg5: 256 x gaussian_problem(512,512,b), QuadraticReg(5e-3 * 1024), fp32
    costs, tol 1e-4 -- per-problem iterations / objective / r_primal of B
    sequential solve()s (solver.cpp:104-241)."""
    from concurrent.futures import ProcessPoolExecutor

    B = 256
    with ProcessPoolExecutor(THREADS) as ex:
        res = list(ex.map(_cfg5_one, range(B)))
    it = np.array([r[0] for r in res], dtype=np.int64)
    obj = np.array([r[1] for r in res])
    rp = np.array([r[2] for r in res])
    term = np.array([r[3] for r in res])
    out = os.path.join(HERE, "full", "full_cfg5_f32.npz")
    np.savez_compressed(out, B=B, m=512, n=512, alpha=5.12, tol=1e-4, iterations=it, objective=obj,
                        r_primal=rp, termination=term)
    print(f"cfg5: mean iterations {it.mean():.1f}, max {it.max()} -> {out}")


def _cfg5_one(b):
    C, p, q, *_ = ora.gaussian_problem(512, 512, b)
    C = C.astype(np.float32).astype(np.float64)
    rep = ora.solve(ora.Problem(C, p, q), ora.quad_reg(5.12), tol_primal=1e-4, max_iter=20000)
    return rep.iterations, rep.objective, rep.r_primal, rep.termination


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES) + ["cfg5_f32"]
    for nm in names:
        if nm == "cfg5_f32":
            run_cfg5()
        else:
            run_case(nm)
