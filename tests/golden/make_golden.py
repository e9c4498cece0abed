#!/usr/bin/env python
"""Regenerates the committed golden fixtures in tests/golden/ (test data, not product code).

The reference (C++, needs Eigen3, absent here -- DESIGN.md §2) cannot be run to
produce golden vectors, and it ships none: its tests draw every
input from a seeded mt19937_64. These fixtures freeze the pinned CPU oracle's
outputs (oracle/otdr_oracle.cpp, checked against the reference's KATs in
tests/test_oracle_kats.py) on small seeded problems, inputs included, so that

  * tests/test_golden.py (CPU) detects any drift of the oracle itself, and
  * tests/test_golden.py (GPU) checks the device path against stored vectors
    that do not depend on the oracle or the data generators at test time.

Each case: inputs (C, p, q[, row labels]), the regularizer, rho =
default_stepsize (solver.cpp:88-93), the state after K raw steps from
make_state (solver.cpp:55-86, :95-102) and a solve() report (solver.cpp:104-241).

  python tests/golden/make_golden.py      # rewrites tests/golden/*.npz
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import pyoracle as ora  # noqa: E402

K = 25

# name: (problem generator, regularizer kind, parameter, solve tolerance)
CASES = {
    # datagen.cpp:56-65 gaussian_problem; alpha = 5e-3 (m + n) as in the configs
    "quad_48x40": (lambda: ora.gaussian_problem(48, 40, 3)[:3] + (None,), "quad", 5e-3 * 88, 1e-6),
    # ragged shape, unregularized DROT (config 2's regularizer)
    "zero_33x57": (lambda: ora.gaussian_problem(33, 57, 4)[:3] + (None,), "none", 0.0, 1e-6),
    # datagen.cpp:67-129 adaptation_problem, 3 classes (config 3's regularizer)
    "gl_60x50": (lambda: (lambda t: (t[0], t[1], t[2], t[5]))(ora.adaptation_problem(60, 50, 3, 5)),
                 "gl", 0.02, 1e-6),
    # test_solver.cpp:393-412 shape: random_problem(Rng(29), 20, 20), 4 row classes
    "gl_random_20x20": (lambda: (lambda r: ora.random_problem(r, 20, 20) + (np.arange(20) % 4,))(ora.Rng(29)),
                        "gl", 0.01, 1e-6),
}


def oracle_reg(kind, param, labels, n):
    if kind == "none":
        return ora.zero_reg()
    if kind == "quad":
        return ora.quad_reg(param)
    offs, cells = ora.column_class_blocks([int(v) for v in labels], n)
    return ora.group_lasso_reg(param, offs, cells)


def make(name):
    gen, kind, param, tol = CASES[name]
    C, p, q, labels = gen()
    m, n = C.shape
    if labels is None:
        labels = np.zeros(m, dtype=np.int32)
    labels = np.asarray(labels, dtype=np.int32)
    reg = oracle_reg(kind, param, labels, n)
    pr = ora.Problem(C, p, q)
    rho = ora.default_stepsize(m, n)
    st = ora.make_state(pr)
    for _ in range(K):
        ora.step(st, pr, reg, rho)
    rep = ora.solve(pr, reg, tol_primal=tol, max_iter=200000)
    return dict(
        C=C, p=p, q=q, labels=labels, kind=np.array(kind), param=np.float64(param),
        rho=np.float64(rho), k=np.int64(st.k), X=st.X, phi=st.phi, psi=st.psi, a=st.a, b=st.b,
        r=st.r, s=st.s, theta=np.float64(st.theta),
        solve_tol=np.float64(tol), solve_iterations=np.int64(rep.iterations),
        solve_termination=np.array(rep.termination), solve_objective=np.float64(rep.objective),
        solve_r_primal=np.float64(rep.r_primal), solve_X=rep.state.X)


def main():
    for name in CASES:
        d = make(name)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **d)
        print(name, d["C"].shape, "k", int(d["k"]), "solve", int(d["solve_iterations"]),
              str(d["solve_termination"]), float(d["solve_objective"]))


if __name__ == "__main__":
    main()
