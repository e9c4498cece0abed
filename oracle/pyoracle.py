"""ctypes binding of the CPU parity oracle (oracle/otdr_oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py -- never by the product package
paper_2305_18483_b200. It exposes the reference's solver API names
(/root/reference/proj/include/otdr/*.hpp) over numpy arrays so the parity tests
read like the reference's own doctest suites.
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libotdr_oracle.so")

OK, E_DIMENSION, E_NEGATIVE, E_MARGINAL, E_ZERO_ITERS, E_INVALID_ARG, E_NONFINITE, E_UNSUPPORTED = range(8)
REG_NONE, REG_QUAD, REG_GROUP_LASSO = 0, 1, 2
TERM_NAMES = {0: "Converged", 1: "MaxIter", 2: "Stalled"}

_dp = ct.POINTER(ct.c_double)
_i32p = ct.POINTER(ct.c_int32)
_i64p = ct.POINTER(ct.c_int64)


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


class _Problem(ct.Structure):
    _fields_ = [("m", ct.c_int64), ("n", ct.c_int64), ("C", _dp), ("p", _dp), ("q", _dp)]


class _Reg(ct.Structure):
    _fields_ = [("kind", ct.c_int), ("param", ct.c_double), ("num_groups", ct.c_int64),
                ("offsets", _i64p), ("cells", _i32p)]


class _State(ct.Structure):
    _fields_ = [("m", ct.c_int64), ("n", ct.c_int64), ("X", _dp), ("phi", _dp), ("psi", _dp),
                ("a", _dp), ("b", _dp), ("r", _dp), ("s", _dp), ("theta", ct.c_double),
                ("eta", ct.c_double), ("k", ct.c_int64)]


class _Options(ct.Structure):
    _fields_ = [("rho", ct.c_double), ("max_iter", ct.c_int64), ("tol_primal", ct.c_double),
                ("has_tol_gap", ct.c_int), ("tol_gap", ct.c_double), ("check_every", ct.c_int64),
                ("deterministic", ct.c_int), ("record_trace", ct.c_int), ("fused", ct.c_int),
                ("threads", ct.c_int)]


class _TraceRow(ct.Structure):
    _fields_ = [("iter", ct.c_int64), ("r_primal", ct.c_double), ("gap", ct.c_double),
                ("dual_residual", ct.c_double), ("support", ct.c_int64), ("elapsed_ms", ct.c_double)]


class _Report(ct.Structure):
    _fields_ = [("objective", ct.c_double), ("iterations", ct.c_int64), ("termination", ct.c_int),
                ("rho", ct.c_double), ("r_primal", ct.c_double),
                ("support_last_change", ct.c_int64), ("trace_len", ct.c_int64)]


_lib = None


def build() -> str:
    """Compile the oracle with its Makefile (test infrastructure)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ct.CDLL(_LIB_PATH)
        L.ora_rng_new.restype = ct.c_void_p
        L.ora_rng_new.argtypes = [ct.c_uint64]
        L.ora_rng_free.argtypes = [ct.c_void_p]
        L.ora_rng_uniform01.restype = ct.c_double
        L.ora_rng_uniform01.argtypes = [ct.c_void_p]
        L.ora_rng_normal.restype = ct.c_double
        L.ora_rng_normal.argtypes = [ct.c_void_p]
        L.ora_rng_raw.restype = ct.c_uint64
        L.ora_rng_raw.argtypes = [ct.c_void_p]
        L.ora_gaussian_problem.argtypes = [ct.c_int64, ct.c_int64, ct.c_uint64, _dp, _dp, _dp, _dp, _dp]
        L.ora_adaptation_problem.argtypes = [ct.c_int64, ct.c_int64, ct.c_int, ct.c_uint64, ct.c_int,
                                             _dp, _dp, _dp, _dp, _dp, _i32p, _i32p]
        L.ora_squared_distance_cost.argtypes = [ct.c_int64, ct.c_int64, ct.c_int64, _dp, _dp, _dp]
        L.ora_validate_problem.argtypes = [ct.c_int64, ct.c_int64, _dp, _dp, _dp, ct.c_char_p, ct.c_int]
        L.ora_normalize_cost.argtypes = [ct.c_int64, ct.c_int64, _dp, ct.POINTER(ct.c_int)]
        L.ora_primal_objective.restype = ct.c_double
        L.ora_primal_objective.argtypes = [ct.POINTER(_Problem), _dp, ct.POINTER(_Reg)]
        L.ora_column_class_blocks.argtypes = [_i32p, ct.c_int64, ct.c_int64, _i32p, _i64p, _i64p]
        L.ora_prox.argtypes = [ct.POINTER(_Reg), ct.c_int64, ct.c_int64, _dp, ct.c_double]
        L.ora_reg_value.restype = ct.c_double
        L.ora_reg_value.argtypes = [ct.POINTER(_Reg), ct.c_int64, ct.c_int64, _dp]
        L.ora_default_stepsize.restype = ct.c_double
        L.ora_default_stepsize.argtypes = [ct.c_int64, ct.c_int64]
        L.ora_default_init.argtypes = [ct.c_int64, ct.c_int64, _dp, _dp]
        L.ora_make_state.argtypes = [ct.POINTER(_Problem), _dp, _dp, _dp, ct.POINTER(_State),
                                     ct.c_char_p, ct.c_int]
        L.ora_step.argtypes = [ct.POINTER(_State), ct.POINTER(_Problem), ct.POINTER(_Reg),
                               ct.c_double, ct.c_int]
        L.ora_solve.argtypes = [ct.POINTER(_Problem), ct.POINTER(_Reg), ct.POINTER(_Options),
                                ct.POINTER(_State), ct.POINTER(_Report), ct.POINTER(_TraceRow),
                                ct.c_int64, ct.c_char_p, ct.c_int]
        L.ora_compute_skip_count.restype = ct.c_int64
        L.ora_compute_skip_count.argtypes = [ct.POINTER(_Problem)]
        L.ora_duality_gap.argtypes = [ct.POINTER(_Problem), ct.POINTER(_Reg), ct.POINTER(_State),
                                      ct.c_double, _dp, _dp, _dp]
        L.ora_dr_reference.argtypes = [ct.POINTER(_Problem), ct.POINTER(_Reg), ct.c_double, _dp,
                                       ct.c_int, _dp, _dp]
        for nm in ("ora_lp_vertex_solve", "ora_transport_simplex"):
            f = getattr(L, nm)
            f.restype = ct.c_int
            f.argtypes = [ct.c_int64, ct.c_int64, _dp, _dp, _dp, _dp, _dp]
        L.ora_affine_project.argtypes = [ct.c_int64, ct.c_int64, _dp, _dp, _dp, _dp]
        L.ora_polytope_project.argtypes = [ct.c_int64, ct.c_int64, _dp, _dp, _dp, ct.c_int, ct.c_double, _dp]
        L.ora_projgrad_solve.restype = ct.c_int
        L.ora_projgrad_solve.argtypes = [ct.c_int64, ct.c_int64, _dp, _dp, _dp, ct.c_double, _dp, _dp]
        _lib = L
    return _lib


def _d(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


# ----------------------------------------------------------------- rng.hpp
class Rng:
    """Seeded mt19937_64 generator (rng.hpp:14-45)."""

    def __init__(self, seed: int):
        self._h = lib().ora_rng_new(ct.c_uint64(seed))

    def uniform01(self) -> float:
        return lib().ora_rng_uniform01(self._h)

    def normal(self) -> float:
        return lib().ora_rng_normal(self._h)

    def raw(self) -> int:
        return lib().ora_rng_raw(self._h)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ora_rng_free(self._h)
            self._h = None


# ----------------------------------------------------------------- datagen
def gaussian_problem(m: int, n: int, seed: int):
    """datagen.cpp:56-65 -> (C, p, q, source_points, target_points)."""
    C = np.empty((m, n)); p = np.empty(m); q = np.empty(n)
    src = np.empty((m, 2)); tgt = np.empty((n, 2))
    lib().ora_gaussian_problem(m, n, seed, _d(C), _d(p), _d(q), _d(src), _d(tgt))
    return C, p, q, src, tgt


def adaptation_problem(m: int, n: int, classes: int, seed: int, identity_map: bool = False):
    """datagen.cpp:67-129 -> (C, p, q, src, tgt, src_labels, tgt_labels)."""
    C = np.empty((m, n)); p = np.empty(m); q = np.empty(n)
    src = np.empty((m, 2)); tgt = np.empty((n, 2))
    ls = np.empty(m, dtype=np.int32); lt = np.empty(n, dtype=np.int32)
    rc = lib().ora_adaptation_problem(m, n, classes, seed, int(identity_map), _d(C), _d(p), _d(q),
                                      _d(src), _d(tgt), ls.ctypes.data_as(_i32p), lt.ctypes.data_as(_i32p))
    if rc:
        raise OracleError(rc, "adaptation_problem arguments")
    return C, p, q, src, tgt, ls, lt


def squared_distance_cost(a, b):
    a = _f64(a); b = _f64(b)
    C = np.empty((a.shape[0], b.shape[0]))
    lib().ora_squared_distance_cost(a.shape[0], b.shape[0], a.shape[1], _d(a), _d(b), _d(C))
    return C


# ----------------------------------------------------------------- problem
def validate_problem(C, p, q):
    C = _f64(C).copy(); p = _f64(p).copy(); q = _f64(q).copy()
    if C.ndim != 2 or C.shape[0] < 1 or C.shape[1] < 1:
        raise OracleError(E_DIMENSION, "cost must be at least 1x1")
    if p.shape[0] != C.shape[0] or q.shape[0] != C.shape[1]:
        raise OracleError(E_DIMENSION, "marginal lengths do not match cost")
    buf = ct.create_string_buffer(512)
    rc = lib().ora_validate_problem(C.shape[0], C.shape[1], _d(C), _d(p), _d(q), buf, 512)
    if rc:
        raise OracleError(rc, buf.value.decode())
    return C, p, q


def normalize_cost(C):
    C = _f64(C).copy()
    z = ct.c_int(0)
    lib().ora_normalize_cost(C.shape[0], C.shape[1], _d(C), ct.byref(z))
    return C, bool(z.value)


# ----------------------------------------------------------------- regs
@dataclass
class Reg:
    """none / quad(alpha) / gl(lambda, CSR groups) -- regularizers.hpp:56-96."""
    kind: int = REG_NONE
    param: float = 0.0
    offsets: np.ndarray | None = None
    cells: np.ndarray | None = None
    _s: _Reg | None = field(default=None, repr=False)

    def struct(self) -> _Reg:
        if self._s is None:
            s = _Reg()
            s.kind = self.kind
            s.param = self.param
            if self.kind == REG_GROUP_LASSO:
                s.num_groups = len(self.offsets) - 1
                s.offsets = self.offsets.ctypes.data_as(_i64p)
                s.cells = self.cells.ctypes.data_as(_i32p)
            self._s = s
        return self._s


def zero_reg() -> Reg:
    return Reg(REG_NONE)


def quad_reg(alpha: float) -> Reg:
    return Reg(REG_QUAD, float(alpha))


def column_class_blocks(labels, n: int):
    """groups.cpp:37-60 -> (offsets int64[G+1], cells int32[T,2])."""
    lab = np.ascontiguousarray(np.asarray(labels, dtype=np.int32))
    m = lab.shape[0]
    cells = np.empty((m * n, 2), dtype=np.int32)
    offs = np.empty(m * n + 1, dtype=np.int64)
    g = ct.c_int64(0)
    rc = lib().ora_column_class_blocks(lab.ctypes.data_as(_i32p), m, n, cells.ctypes.data_as(_i32p),
                                       offs.ctypes.data_as(_i64p), ct.byref(g))
    if rc:
        raise OracleError(rc, "column_class_blocks: bad labels")
    return offs[: g.value + 1].copy(), cells[: offs[g.value]].copy()


def group_lasso_reg(lam: float, offsets, cells) -> Reg:
    return Reg(REG_GROUP_LASSO, float(lam), np.ascontiguousarray(offsets, dtype=np.int64),
               np.ascontiguousarray(cells, dtype=np.int32))


def prox(reg: Reg, V, rho: float):
    V = _f64(V).copy()
    lib().ora_prox(ct.byref(reg.struct()), V.shape[0], V.shape[1], _d(V), rho)
    return V


def reg_value(reg: Reg, X) -> float:
    X = _f64(X)
    return lib().ora_reg_value(ct.byref(reg.struct()), X.shape[0], X.shape[1], _d(X))


# ----------------------------------------------------------------- solver
class Problem:
    def __init__(self, C, p, q):
        self.C = _f64(C); self.p = _f64(p); self.q = _f64(q)
        self.m, self.n = self.C.shape
        self._s = _Problem(self.m, self.n, _d(self.C), _d(self.p), _d(self.q))

    def struct(self):
        return self._s


class State:
    """SolverState (solver.hpp:51-59) over numpy arrays."""

    def __init__(self, m: int, n: int):
        self.X = np.zeros((m, n)); self.phi = np.zeros(m); self.psi = np.zeros(n)
        self.a = np.zeros(m); self.b = np.zeros(n); self.r = np.zeros(m); self.s = np.zeros(n)
        self._s = _State(m, n, _d(self.X), _d(self.phi), _d(self.psi), _d(self.a), _d(self.b),
                         _d(self.r), _d(self.s), 0.0, 0.0, 0)

    theta = property(lambda self: self._s.theta)
    eta = property(lambda self: self._s.eta)
    k = property(lambda self: self._s.k)

    def struct(self):
        return self._s

    def shadow(self):
        return self.X + self.phi[:, None] + self.psi[None, :]


def default_stepsize(m: int, n: int) -> float:
    return lib().ora_default_stepsize(m, n)


def default_init(m: int, n: int):
    phi = np.empty(m); psi = np.empty(n)
    lib().ora_default_init(m, n, _d(phi), _d(psi))
    return np.zeros((m, n)), phi, psi


def make_state(pr: Problem, init=None) -> State:
    st = State(pr.m, pr.n)
    buf = ct.create_string_buffer(256)
    if init is None:
        rc = lib().ora_make_state(ct.byref(pr.struct()), None, None, None, ct.byref(st.struct()), buf, 256)
    else:
        X0, phi0, psi0 = (_f64(v) for v in init)
        if X0.shape != (pr.m, pr.n) or phi0.shape != (pr.m,) or psi0.shape != (pr.n,):
            raise OracleError(E_DIMENSION, "warm start dimensions do not match the problem")
        rc = lib().ora_make_state(ct.byref(pr.struct()), _d(X0), _d(phi0), _d(psi0),
                                  ct.byref(st.struct()), buf, 256)
    if rc:
        raise OracleError(rc, buf.value.decode())
    return st


def step(st: State, pr: Problem, reg: Reg, rho: float, threads: int = 1) -> None:
    lib().ora_step(ct.byref(st.struct()), ct.byref(pr.struct()), ct.byref(reg.struct()), rho, threads)


@dataclass
class Report:
    state: State
    objective: float
    iterations: int
    termination: str
    rho: float
    r_primal: float
    support_last_change: int
    trace: list


def solve(pr: Problem, reg: Reg, rho=0.0, max_iter=100000, tol_primal=1e-4, tol_gap=None,
          check_every=1, deterministic=False, record_trace=False, fused=False, init=None,
          threads=1, trace_cap=100000) -> Report:
    st = make_state(pr, init)
    opt = _Options(rho, max_iter, tol_primal, int(tol_gap is not None),
                   0.0 if tol_gap is None else tol_gap, check_every, int(deterministic),
                   int(record_trace), int(fused), threads)
    rep = _Report()
    cap = trace_cap if record_trace else 0
    rows = (_TraceRow * max(cap, 1))()
    buf = ct.create_string_buffer(256)
    rc = lib().ora_solve(ct.byref(pr.struct()), ct.byref(reg.struct()), ct.byref(opt),
                         ct.byref(st.struct()), ct.byref(rep), rows, cap, buf, 256)
    if rc:
        raise OracleError(rc, buf.value.decode())
    trace = [(r.iter, r.r_primal, r.gap, r.dual_residual, r.support, r.elapsed_ms)
             for r in rows[: min(rep.trace_len, cap)]]
    return Report(st, rep.objective, rep.iterations, TERM_NAMES[rep.termination], rep.rho,
                  rep.r_primal, rep.support_last_change, trace)


def primal_objective(pr: Problem, X, reg: Reg) -> float:
    X = _f64(X)
    return lib().ora_primal_objective(ct.byref(pr.struct()), _d(X), ct.byref(reg.struct()))


def compute_skip_count(pr: Problem) -> int:
    return lib().ora_compute_skip_count(ct.byref(pr.struct()))


def duality_gap(pr: Problem, reg: Reg, st: State, rho: float):
    dv, gap, dres = ct.c_double(), ct.c_double(), ct.c_double()
    lib().ora_duality_gap(ct.byref(pr.struct()), ct.byref(reg.struct()), ct.byref(st.struct()), rho,
                          ct.byref(dv), ct.byref(gap), ct.byref(dres))
    return dv.value, gap.value, dres.value


def dr_reference(pr: Problem, reg: Reg, rho: float, y0, iters: int):
    y0 = _f64(y0)
    xs = np.empty((iters, pr.m, pr.n)); ys = np.empty((iters, pr.m, pr.n))
    lib().ora_dr_reference(ct.byref(pr.struct()), ct.byref(reg.struct()), rho, _d(y0), iters, _d(xs), _d(ys))
    return xs, ys


def random_problem(rng: Rng, m: int, n: int, cost_floor: float = 0.0):
    """The tests' local helper (test_solver.cpp:19-29): draws C, p, q from rng."""
    C = np.empty((m, n))
    for i in range(m):
        for j in range(n):
            C[i, j] = cost_floor + rng.uniform01()
    p = np.array([rng.uniform01() + 0.05 for _ in range(m)])
    q = np.array([rng.uniform01() + 0.05 for _ in range(n)])
    p = p / p.sum()
    q = q / q.sum()
    return validate_problem(C, p, q)


# ----------------------------------------------------------------- optimality oracles
# (tests/support/oracles.cpp:16-345 -- answers that do not come from DR)
def affine_project(Z, p, q):
    Z = _f64(Z); p = _f64(p); q = _f64(q)
    out = np.empty_like(Z)
    lib().ora_affine_project(Z.shape[0], Z.shape[1], _d(Z), _d(p), _d(q), _d(out))
    return out


def polytope_project(Z, p, q, max_iter=500000, tol=1e-13):
    Z = _f64(Z); p = _f64(p); q = _f64(q)
    out = np.empty_like(Z)
    lib().ora_polytope_project(Z.shape[0], Z.shape[1], _d(Z), _d(p), _d(q), max_iter, tol, _d(out))
    return out


def _lp(fn, C, p, q):
    C = _f64(C); p = _f64(p); q = _f64(q)
    X = np.empty_like(C)
    v = ct.c_double()
    rc = fn(C.shape[0], C.shape[1], _d(C), _d(p), _d(q), _d(X), ct.byref(v))
    if rc:
        raise OracleError(rc, "LP oracle failed")
    return X, v.value


def lp_vertex_solve(C, p, q):
    """Exact LP by spanning-tree basis enumeration (oracles.cpp:164-211): (plan, value)."""
    return _lp(lib().ora_lp_vertex_solve, C, p, q)


def transport_simplex(C, p, q):
    """Transportation simplex, Bland's rule (oracles.cpp:213-345): (plan, value)."""
    return _lp(lib().ora_transport_simplex, C, p, q)


def projgrad_solve(C, p, q, alpha):
    """argmin <C,X> + alpha/2 ||X||^2 over the transport polytope (oracles.cpp:73-101)."""
    C = _f64(C); p = _f64(p); q = _f64(q)
    X = np.empty_like(C)
    gm = ct.c_double()
    rc = lib().ora_projgrad_solve(C.shape[0], C.shape[1], _d(C), _d(p), _d(q), float(alpha), _d(X),
                                  ct.byref(gm))
    if rc:
        raise OracleError(rc, f"projgrad_solve: gradient mapping {gm.value}")
    return X


def small_suite_problem(sd: int):
    """acceptance_main.cpp:33-38: seeds 2000+sd, sides 2..4 drawn from the rng."""
    rng = Rng(2000 + sd)
    m = 2 + int(rng.uniform01() * 3.0)
    n = 2 + int(rng.uniform01() * 3.0)
    return random_problem(rng, m, n)
