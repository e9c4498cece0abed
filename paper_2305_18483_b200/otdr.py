"""Host-side mirror of the reference solver API (proj/include/otdr/*.hpp) over
the B200 C-ABI (include/otdr_dev.h).

Names, argument meaning and error behaviour follow the reference:

    validate_problem / normalize_cost / primal_objective   problem.hpp:24-33
    ZeroReg / QuadraticReg / GroupLassoReg                 regularizers.hpp:56-96
    make_partition / column_class_blocks                   groups.hpp:30-34
    default_stepsize / default_init / make_state / step /  solver.hpp:89-108
    solve / compute_skip_count
    recover_duals / duality_gap / ot_cost_gradient         duality.hpp:27-39
    DimensionMismatch, NegativeEntry, ...                  errors.hpp:9-34

Every plan-sized operation (the DR iteration, the stopping logic, the objective
and the duality certificate) runs in the sm_100a kernels of libotdr_dev.so;
there is no CPU fallback. Host code here only validates inputs, moves buffers
and maps status codes to the reference's exception types.

Storage: `SolverOptions.storage` selects how C and X live in HBM. "f64"
(default for this API) reproduces the reference's element-wise rounding; "f32"
halves the bytes per iteration (arithmetic stays fp64 in registers).
"""
from __future__ import annotations

import ctypes as ct
import enum
import math
from dataclasses import dataclass, field
from typing import NamedTuple, Optional

import numpy as np

from . import _native as nat

# ----------------------------------------------------------------- errors.hpp


class OtdrError(Exception):
    """Base of every error raised by the B200 backend."""


class DimensionMismatch(OtdrError, ValueError):  # errors.hpp:10
    pass


class NegativeEntry(OtdrError, ValueError):  # errors.hpp:13
    pass


class MarginalSumOutOfRange(OtdrError, ValueError):  # errors.hpp:16
    pass


class ZeroIterations(OtdrError, ValueError):  # errors.hpp:19
    pass


class InvalidArgument(OtdrError, ValueError):  # std::invalid_argument
    pass


class NonFiniteIterate(OtdrError, RuntimeError):  # errors.hpp:26
    pass


class Unsupported(OtdrError, NotImplementedError):
    """A regularizer or group partition the B200 kernels do not cover."""


class DeviceError(OtdrError, RuntimeError):
    """CUDA / NCCL failure (including: no CUDA device)."""


_ERRORS = {1: DimensionMismatch, 2: NegativeEntry, 3: MarginalSumOutOfRange, 4: ZeroIterations,
           5: InvalidArgument, 6: NonFiniteIterate, 7: Unsupported, 8: DeviceError, 9: DeviceError,
           10: InvalidArgument}

_STORAGE = {"f32": nat.STORE_F32, "f64": nat.STORE_F64}


def _f64(a, shape=None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None and a.shape != shape:
        raise DimensionMismatch(f"expected shape {shape}, got {a.shape}")
    return a


# ---------------------------------------------------------------- problem.hpp
@dataclass
class Problem:
    """min <C,X> + h(X) s.t. X1 = p, X^T 1 = q, X >= 0 (problem.hpp:13-21)."""
    cost: np.ndarray
    p: np.ndarray
    q: np.ndarray
    _engines: dict = field(default_factory=dict, repr=False, compare=False)

    def rows(self) -> int:
        return self.cost.shape[0]

    def cols(self) -> int:
        return self.cost.shape[1]


_REJECT_TOL = 1e-6   # problem.cpp:15
_SKIP_TOL = 1e-13    # problem.cpp:18


def _check_marginal(v: np.ndarray, which: str) -> None:
    bad = ~(np.isfinite(v) & (v >= 0.0))
    if bad.any():
        i = int(np.argmax(bad))
        raise NegativeEntry(f"{which}[{i}] must be finite and >= 0, got {v[i]}")
    s = float(np.sum(v))
    if abs(s - 1.0) > _REJECT_TOL:
        raise MarginalSumOutOfRange(f"{which} sums to {s:f}, more than 1e-6 away from 1")


def validate_problem(cost, p, q) -> Problem:
    """problem.cpp:41-66: dimensions, signs, marginals renormalized within 1e-6."""
    cost = np.array(cost, dtype=np.float64, copy=True, order="C")
    p = np.array(p, dtype=np.float64, copy=True).reshape(-1)
    q = np.array(q, dtype=np.float64, copy=True).reshape(-1)
    if cost.ndim != 2 or cost.shape[0] < 1 or cost.shape[1] < 1:
        raise DimensionMismatch("cost must be at least 1x1")
    if p.shape[0] != cost.shape[0] or q.shape[0] != cost.shape[1]:
        raise DimensionMismatch(f"marginal lengths ({p.shape[0]}, {q.shape[0]}) do not match cost "
                                f"{cost.shape[0]}x{cost.shape[1]}")
    bad = ~(np.isfinite(cost) & (cost >= 0.0))
    if bad.any():
        i, j = np.unravel_index(int(np.argmax(bad)), cost.shape)
        raise NegativeEntry(f"cost({i},{j}) must be finite and >= 0, got {cost[i, j]}")
    _check_marginal(p, "p")
    _check_marginal(q, "q")
    for v in (p, q):
        s = float(np.sum(v))
        if abs(s - 1.0) > _SKIP_TOL:
            v /= s
    return Problem(cost, p, q)


def normalize_cost(problem: Problem, return_all_zero: bool = False):
    """problem.cpp:68-74: divide C by its max entry (all-zero cost unchanged)."""
    mx = float(problem.cost.max())
    zero = not (mx > 0.0)
    cost = problem.cost if zero else problem.cost / mx
    out = Problem(np.ascontiguousarray(cost), problem.p.copy(), problem.q.copy())
    return (out, zero) if return_all_zero else out


# ----------------------------------------------------------------- groups.hpp
@dataclass
class GroupPartition:
    """Disjoint CSR groups of (row, col) cells (groups.hpp:15-27)."""
    rows: int
    cols: int
    cells: np.ndarray    # (T, 2) int32
    offsets: np.ndarray  # (G + 1,) int64
    row_labels: Optional[np.ndarray] = None  # set when built by column_class_blocks

    def num_groups(self) -> int:
        return len(self.offsets) - 1

    def group(self, g: int) -> np.ndarray:
        return self.cells[self.offsets[g]:self.offsets[g + 1]]


def make_partition(rows: int, cols: int, groups) -> GroupPartition:
    """groups.cpp:8-35: bounds and disjointness checks (InvalidArgument)."""
    seen = np.zeros((rows, cols), dtype=bool)
    cells, offsets = [], [0]
    for grp in groups:
        for (i, j) in grp:
            if i < 0 or i >= rows or j < 0 or j >= cols:
                raise InvalidArgument(f"group cell ({i},{j}) outside {rows}x{cols} grid")
            if seen[i, j]:
                raise InvalidArgument(f"group cell ({i},{j}) appears in more than one group")
            seen[i, j] = True
            cells.append((i, j))
        offsets.append(len(cells))
    return GroupPartition(rows, cols, np.array(cells, dtype=np.int32).reshape(-1, 2),
                          np.array(offsets, dtype=np.int64))


def column_class_blocks(row_labels, cols: int) -> GroupPartition:
    """groups.cpp:37-60: one group per (column, present class), column-major."""
    lab = np.asarray(row_labels, dtype=np.int64).reshape(-1)
    if lab.size == 0:
        raise InvalidArgument("no row labels")
    if cols < 1:
        raise InvalidArgument("need at least one column")
    if (lab < 0).any():
        raise InvalidArgument("row labels must be >= 0")
    classes = [c for c in range(int(lab.max()) + 1) if (lab == c).any()]
    rows_of = [np.nonzero(lab == c)[0] for c in classes]
    per_col = np.concatenate(rows_of) if rows_of else np.zeros(0, dtype=np.int64)
    sizes = np.array([len(r) for r in rows_of], dtype=np.int64)
    cells = np.empty((cols * per_col.size, 2), dtype=np.int32)
    cells[:, 0] = np.tile(per_col, cols)
    cells[:, 1] = np.repeat(np.arange(cols), per_col.size)
    offsets = np.concatenate([[0], np.cumsum(np.tile(sizes, cols))]).astype(np.int64)
    return GroupPartition(int(lab.size), int(cols), cells, offsets, lab.astype(np.int32))


def _labels_of(part: GroupPartition) -> np.ndarray:
    """Row labels (-1 = uncovered) of a column_class_blocks-shaped partition.

    The kernels cover partitions where every group lies in one column and all
    columns split their rows into the same row sets; anything else raises
    Unsupported (no CPU fallback)."""
    if part.row_labels is not None:
        return part.row_labels
    G = part.num_groups()
    if G == 0:
        return np.full(part.rows, -1, dtype=np.int32)
    sizes = np.diff(part.offsets)
    gid = np.repeat(np.arange(G), sizes)
    c = part.cells
    cmin = np.minimum.reduceat(c[:, 1], part.offsets[:-1][sizes > 0]) if c.size else np.zeros(0)
    cmax = np.maximum.reduceat(c[:, 1], part.offsets[:-1][sizes > 0]) if c.size else np.zeros(0)
    if (cmin != cmax).any():
        raise Unsupported("group spans several columns: not a column_class_blocks partition")
    lab = np.full((part.rows, part.cols), -1, dtype=np.int64)
    lab[c[:, 0], c[:, 1]] = gid
    base = lab[:, 0]
    # canonical class id per row: order of first appearance in column 0
    canon = np.full(part.rows, -1, dtype=np.int32)
    ids = {}
    for i, g in enumerate(base):
        if g >= 0:
            canon[i] = ids.setdefault(int(g), len(ids))
    for j in range(part.cols):
        col = lab[:, j]
        if ((col < 0) != (base < 0)).any():
            raise Unsupported("columns cover different rows: not a column_class_blocks partition")
        pairs = {}
        for i in np.nonzero(col >= 0)[0]:
            if pairs.setdefault(int(col[i]), canon[i]) != canon[i]:
                raise Unsupported("row sets differ across columns: not column_class_blocks")
        if len(set(pairs.values())) != len(pairs):
            raise Unsupported("row sets differ across columns: not column_class_blocks")
    return canon


# ---------------------------------------------------------- regularizers.hpp
class Regularizer:
    """Regularizer selection for the device kernels (regularizers.hpp:29-53).

    The prox runs inside the fused sweep kernel; value() goes through the
    device objective kernel."""
    kind = nat.REG_NONE
    param = 0.0

    def name(self) -> str:
        raise NotImplementedError

    def _labels(self, rows: int):
        return None


class ZeroReg(Regularizer):  # regularizers.hpp:56-61
    kind = nat.REG_NONE

    def name(self) -> str:
        return "none"


class QuadraticReg(Regularizer):  # regularizers.hpp:63-79
    kind = nat.REG_QUAD

    def __init__(self, alpha: float):
        if not (alpha > 0.0) or not math.isfinite(alpha):
            raise InvalidArgument("quadratic regularizer needs alpha > 0")
        self.param = float(alpha)

    def alpha(self) -> float:
        return self.param

    def name(self) -> str:
        return f"quad:alpha={self.param:g}"


class GroupLassoReg(Regularizer):  # regularizers.hpp:81-96
    kind = nat.REG_GROUP_LASSO

    def __init__(self, lambda_: float, partition: GroupPartition):
        if not (lambda_ > 0.0) or not math.isfinite(lambda_):
            raise InvalidArgument("group lasso needs lambda > 0")
        self.param = float(lambda_)
        self._partition = partition
        self._row_labels = None

    def lambda_(self) -> float:
        return self.param

    def partition(self) -> GroupPartition:
        return self._partition

    def name(self) -> str:
        return f"gl:lambda={self.param:g}"

    def _labels(self, rows: int):
        if self._row_labels is None:
            if self._partition.rows != rows:
                raise DimensionMismatch("group partition rows do not match the problem")
            self._row_labels = np.ascontiguousarray(_labels_of(self._partition), dtype=np.int32)
        return self._row_labels


# --------------------------------------------------------------- solver.hpp
class Termination(enum.Enum):  # solver.hpp:61
    Converged = 0
    MaxIter = 1
    Stalled = 2


def to_string(t: Termination) -> str:
    return t.name


@dataclass
class WarmStart:  # solver.hpp:34-37
    plan0: np.ndarray
    phi0: np.ndarray
    psi0: np.ndarray


@dataclass
class SolverOptions:  # solver.hpp:39-49 (+ storage / device extensions)
    rho: float = 0.0
    max_iter: int = 100000
    tol_primal: float = 1e-4
    tol_gap: Optional[float] = None
    check_every: int = 1
    deterministic: bool = False
    record_trace: bool = False
    fused: bool = False
    init: Optional[WarmStart] = None
    storage: str = "f64"
    device: int = 0


@dataclass
class SolverState:  # solver.hpp:51-59
    X: np.ndarray
    phi: np.ndarray
    psi: np.ndarray
    a: np.ndarray
    b: np.ndarray
    theta: float
    r: np.ndarray
    s: np.ndarray
    eta: float
    k: int


class TraceRow(NamedTuple):  # solver.hpp:65-72
    iter: int
    r_primal: float
    gap: float
    dual_residual: float
    support: int
    elapsed_ms: float


@dataclass
class SolveReport:  # solver.hpp:74-87
    state: Optional[SolverState]
    objective: float
    iterations: int
    termination: Termination
    rho: float
    r_primal: float
    trace: list
    support_last_change: int
    device_ms: float = 0.0

    def plan(self) -> np.ndarray:
        return self.state.X


@dataclass
class DualCertificate:  # duality.hpp:19-24
    mu: np.ndarray
    nu: np.ndarray
    dual_value: float
    gap: float
    dual_residual: float


@dataclass
class Shard:
    """Row band of a row-sharded multi-GPU run (one process per GPU)."""
    rank: int
    nranks: int
    row_begin: int
    row_end: int
    nccl_id: Optional[bytes] = None  # None: exchange over peer memory only (Engine.peer_*)


def default_stepsize(m: int, n: int) -> float:  # solver.cpp:55-57
    return 2.0 / float(m + n)


def default_init(m: int, n: int) -> WarmStart:  # solver.cpp:59-66
    mn = float(m + n)
    return WarmStart(np.zeros((m, n)), np.full(m, (1.0 + m / mn) / (3.0 * mn)),
                     np.full(n, (1.0 + n / mn) / (3.0 * mn)))


# ------------------------------------------------------------------ engine
class Engine:
    """One device context (libotdr_dev.so) holding C, X and the DR state in HBM.

    The reference-shaped functions below drive an Engine; callers that want
    the raw speed (bench, batched loops) use it directly."""

    def __init__(self, m: int, n: int, storage: str = "f32", device: int = 0,
                 shard: Optional[Shard] = None):
        self._L = nat.lib()
        cfg = nat.DevConfig()
        cfg.device = device
        cfg.storage = _STORAGE[storage]
        cfg.m, cfg.n = m, n
        if shard is None:
            cfg.rank, cfg.nranks, cfg.row_begin, cfg.row_end, cfg.nccl_id = 0, 1, 0, m, None
            self.row_begin, self.row_end = 0, m
        else:
            cfg.rank, cfg.nranks = shard.rank, shard.nranks
            cfg.row_begin, cfg.row_end = shard.row_begin, shard.row_end
            cfg.nccl_id = shard.nccl_id
            self.row_begin, self.row_end = shard.row_begin, shard.row_end
        self.m, self.n, self.storage = m, n, storage
        self.m_local = self.row_end - self.row_begin
        h = ct.c_void_p()
        rc = self._L.otdr_dev_create(ct.byref(cfg), ct.byref(h))
        if rc != nat.OTDR_OK:
            raise _ERRORS.get(rc, DeviceError)(
                f"otdr_dev_create failed ({nat.STATUS_NAMES.get(rc, rc)})")
        self._h = h
        self._reg_key = None

    def close(self):
        if getattr(self, "_h", None):
            self._L.otdr_dev_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ck(self, rc: int):
        if rc != nat.OTDR_OK:
            msg = self._L.otdr_dev_last_error(self._h).decode(errors="replace")
            raise _ERRORS.get(rc, DeviceError)(msg or nat.STATUS_NAMES.get(rc, str(rc)))

    # -- problem / regularizer / state
    def set_problem(self, cost_local, p_local, q):
        C = _f64(cost_local, (self.m_local, self.n))
        p = _f64(p_local, (self.m_local,))
        q = _f64(q, (self.n,))
        self._ck(self._L.otdr_dev_set_problem(self._h, nat.dptr(C), nat.dptr(p), nat.dptr(q)))

    def read_cost_otpb(self, path: str, p_local, q):
        """Load this engine's rows of an OTPB cost file (io.cpp:127-158) into HBM."""
        p = _f64(p_local, (self.m_local,))
        q = _f64(q, (self.n,))
        self._ck(self._L.otdr_dev_read_cost_otpb(self._h, str(path).encode(), nat.dptr(p), nat.dptr(q)))

    def write_plan_otpb(self, path: str):
        """Write the plan (this engine's rows) as OTPB straight from HBM."""
        self._ck(self._L.otdr_dev_write_plan_otpb(self._h, str(path).encode()))

    def build_sqdist_cost(self, src_local, tgt, p_local, q) -> bool:
        src = _f64(src_local)
        tgt = _f64(tgt)
        p = _f64(p_local, (self.m_local,))
        q = _f64(q, (self.n,))
        z = ct.c_int(0)
        self._ck(self._L.otdr_dev_build_sqdist_cost(self._h, nat.dptr(src), nat.dptr(tgt),
                                                    src.shape[1], nat.dptr(p), nat.dptr(q),
                                                    ct.byref(z)))
        return bool(z.value)

    def set_regularizer(self, reg: Regularizer, labels_local=None):
        if not isinstance(reg, (ZeroReg, QuadraticReg, GroupLassoReg)):
            raise Unsupported(f"regularizer {type(reg).__name__} has no B200 kernel")
        lab = None
        if reg.kind == nat.REG_GROUP_LASSO:
            lab = labels_local if labels_local is not None else reg._labels(self.m)[
                self.row_begin:self.row_end]
            lab = np.ascontiguousarray(lab, dtype=np.int32)
        key = (reg.kind, reg.param, None if lab is None else lab.tobytes())
        if key == self._reg_key:
            return
        ptr = None if lab is None else lab.ctypes.data_as(ct.POINTER(ct.c_int32))
        self._ck(self._L.otdr_dev_set_regularizer(self._h, reg.kind, reg.param, ptr))
        self._reg_key = key

    def set_state(self, init: Optional[WarmStart] = None):
        if init is None:
            self._ck(self._L.otdr_dev_set_state(self._h, None, None, None))
            return
        X0 = _f64(init.plan0)
        phi0 = _f64(init.phi0).reshape(-1)
        psi0 = _f64(init.psi0).reshape(-1)
        if X0.shape != (self.m_local, self.n) or phi0.shape != (self.m_local,) or \
                psi0.shape != (self.n,):
            raise DimensionMismatch("warm start dimensions do not match the problem")
        self._ck(self._L.otdr_dev_set_state(self._h, nat.dptr(X0), nat.dptr(phi0), nat.dptr(psi0)))

    def load_state(self, st: SolverState):
        arrs = [_f64(st.X, (self.m_local, self.n)), _f64(st.phi, (self.m_local,)),
                _f64(st.psi, (self.n,)), _f64(st.a, (self.m_local,)), _f64(st.b, (self.n,)),
                _f64(st.r, (self.m_local,)), _f64(st.s, (self.n,))]
        self._ck(self._L.otdr_dev_load_state(self._h, *[nat.dptr(a) for a in arrs],
                                             float(st.theta), float(st.eta), int(st.k)))

    def get_state(self, with_plan: bool = True) -> SolverState:
        ml, n = self.m_local, self.n
        X = np.empty((ml, n)) if with_plan else None
        phi, a, r = np.empty(ml), np.empty(ml), np.empty(ml)
        psi, b, s = np.empty(n), np.empty(n), np.empty(n)
        th, et, k = ct.c_double(), ct.c_double(), ct.c_int64()
        self._ck(self._L.otdr_dev_get_state(self._h, nat.dptr(X), nat.dptr(phi), nat.dptr(psi),
                                            nat.dptr(a), nat.dptr(b), nat.dptr(r), nat.dptr(s),
                                            ct.byref(th), ct.byref(et), ct.byref(k)))
        return SolverState(X, phi, psi, a, b, th.value, r, s, et.value, k.value)

    def get_plan_into(self, out: np.ndarray):
        """Download X into a caller-owned (e.g. pinned) fp64 buffer."""
        self._ck(self._L.otdr_dev_get_state(self._h, nat.dptr(out), None, None, None, None, None,
                                            None, None, None, None))

    # -- iteration
    def step(self, rho: float, iters: int = 1):
        self._ck(self._L.otdr_dev_step(self._h, float(rho), int(iters)))

    def solve(self, opt: SolverOptions, with_state: bool = True) -> SolveReport:
        o = nat.SolveOpts()
        o.rho = opt.rho
        o.max_iter = int(opt.max_iter)
        o.tol_primal = opt.tol_primal
        o.has_tol_gap = 0 if opt.tol_gap is None else 1
        o.tol_gap = 0.0 if opt.tol_gap is None else float(opt.tol_gap)
        o.check_every = int(opt.check_every)
        o.deterministic = int(bool(opt.deterministic))
        o.record_trace = int(bool(opt.record_trace))
        o.fused = int(bool(opt.fused))
        res = nat.SolveResult()
        self._ck(self._L.otdr_dev_solve(self._h, ct.byref(o), ct.byref(res)))
        trace = []
        if opt.record_trace and res.trace_rows > 0:
            rows = (nat.TraceRow * res.trace_rows)()
            cnt = ct.c_int64()
            self._ck(self._L.otdr_dev_get_trace(self._h, rows, res.trace_rows, ct.byref(cnt)))
            trace = [TraceRow(r.iter, r.r_primal, r.gap, r.dual_residual, r.support, r.elapsed_ms)
                     for r in rows[:cnt.value]]
        st = self.get_state() if with_state else None
        return SolveReport(st, res.objective, res.iterations, Termination(res.termination),
                           res.rho, res.r_primal, trace, res.support_last_change, res.device_ms)

    def objective(self) -> float:
        out = ct.c_double()
        self._ck(self._L.otdr_dev_objective(self._h, ct.byref(out)))
        return out.value

    def duality_gap(self, rho: float):
        c = nat.Certificate()
        self._ck(self._L.otdr_dev_duality_gap(self._h, float(rho), ct.byref(c)))
        return c.dual_value, c.gap, c.dual_residual

    # -- measurement
    def profile(self, rho: float, iters: int) -> dict:
        t = nat.KernelTimes()
        self._ck(self._L.otdr_dev_profile(self._h, float(rho), int(iters), ct.byref(t)))
        return {"sweep_ms": t.sweep_ms, "reduce_ms": t.reduce_ms, "exchange_ms": t.exchange_ms,
                "update_ms": t.update_ms, "iterations": t.iterations, "sweep_bytes": t.sweep_bytes}

    def time_steps(self, rho: float, iters: int) -> float:
        ms = ct.c_double()
        self._ck(self._L.otdr_dev_time_steps(self._h, float(rho), int(iters), ct.byref(ms)))
        return ms.value

    # -- peer-memory exchange of row-sharded runs (CUDA IPC over NVLink)
    def peer_export(self) -> bytes:
        """This rank's receive-buffer IPC handle (all-gather it across ranks)."""
        buf = ct.create_string_buffer(nat.PEER_HANDLE_BYTES)
        self._ck(self._L.otdr_dev_peer_export(self._h, buf))
        return buf.raw

    def peer_import(self, handles) -> None:
        """Open every rank's handle (rank order); the solve loop then exchanges
        column sums over peer memory inside the streaming kernel."""
        blob = b"".join(handles)
        self._ck(self._L.otdr_dev_peer_import(self._h, blob))

    def kernels_per_iteration(self) -> int:
        """Launches per DR iteration on the graph path; 0 for persistent loops."""
        return self._L.otdr_dev_kernels_per_iteration(self._h)

    def solve_path(self) -> str:
        """Device loop used by step()/solve(): "graph", "resident" or "stream"."""
        return ("graph", "resident", "stream")[self._L.otdr_dev_solve_path(self._h)]

    def kernel_name(self) -> str:
        """The kernel step()/solve() launch in the current configuration."""
        return self._L.otdr_dev_kernel_name(self._h).decode()


def link_local(engines) -> None:
    """Link the rank contexts of ONE process (engines[r] = rank r) for the
    peer-memory exchange -- the multi-rank path on one GPU (tests)."""
    L = nat.lib()
    arr = (ct.c_void_p * len(engines))(*[e._h for e in engines])
    rc = L.otdr_dev_peer_link_local(arr, len(engines))
    if rc != nat.OTDR_OK:
        msg = L.otdr_dev_last_error(engines[0]._h).decode(errors="replace")
        raise _ERRORS.get(rc, DeviceError)(msg or nat.STATUS_NAMES.get(rc, str(rc)))


class BatchEngine:
    """B same-shape problems solved by one launch (libotdr_dev.so otdr_batch_*):
    each problem's C and X stay resident in a thread-block cluster's shared
    memory for the whole solve. Equivalent to B sequential `solve()` calls from
    `default_init` -- the GAN minibatch loop of the paper."""

    def __init__(self, batch: int, m: int, n: int, storage: str = "f32", device: int = 0):
        self._L = nat.lib()
        self.batch, self.m, self.n, self.storage = batch, m, n, storage
        h = ct.c_void_p()
        rc = self._L.otdr_batch_create(device, _STORAGE[storage], batch, m, n, ct.byref(h))
        if rc != nat.OTDR_OK:
            raise _ERRORS.get(rc, DeviceError)(
                f"otdr_batch_create failed ({nat.STATUS_NAMES.get(rc, rc)})")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            self._L.otdr_batch_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ck(self, rc: int):
        if rc != nat.OTDR_OK:
            msg = self._L.otdr_batch_last_error(self._h).decode(errors="replace")
            raise _ERRORS.get(rc, DeviceError)(msg or nat.STATUS_NAMES.get(rc, str(rc)))

    def set_problems(self, costs, p, q):
        B, m, n = self.batch, self.m, self.n
        C = _f64(costs, (B, m, n))
        self._ck(self._L.otdr_batch_set_problems(self._h, nat.dptr(C), nat.dptr(_f64(p, (B, m))),
                                                 nat.dptr(_f64(q, (B, n)))))

    def build_sqdist_costs(self, src, tgt, p, q):
        B, m, n = self.batch, self.m, self.n
        s = _f64(src)
        t = _f64(tgt)
        if s.shape[:2] != (B, m) or t.shape[:2] != (B, n) or s.shape[2] != t.shape[2]:
            raise DimensionMismatch("point clouds do not match the batch shape")
        self._ck(self._L.otdr_batch_build_sqdist_costs(self._h, nat.dptr(s), nat.dptr(t), s.shape[2],
                                                       nat.dptr(_f64(p, (B, m))),
                                                       nat.dptr(_f64(q, (B, n)))))

    def set_regularizer(self, reg: Regularizer):
        if not isinstance(reg, (ZeroReg, QuadraticReg)):
            raise Unsupported("the batched entry point covers zero / quadratic regularizers")
        self._ck(self._L.otdr_batch_set_regularizer(self._h, reg.kind, reg.param))

    def solve(self, opt: SolverOptions) -> list:
        o = nat.SolveOpts(opt.rho, int(opt.max_iter), opt.tol_primal, int(opt.tol_gap is not None),
                          0.0 if opt.tol_gap is None else float(opt.tol_gap), int(opt.check_every),
                          int(bool(opt.deterministic)), int(bool(opt.record_trace)),
                          int(bool(opt.fused)))
        res = (nat.SolveResult * self.batch)()
        self._ck(self._L.otdr_batch_solve(self._h, ct.byref(o), res))
        return [SolveReport(None, r.objective, r.iterations, Termination(r.termination), r.rho,
                            r.r_primal, [], -1, r.device_ms) for r in res]

    def plans(self):
        B, m, n = self.batch, self.m, self.n
        X = np.empty((B, m, n))
        phi = np.empty((B, m))
        psi = np.empty((B, n))
        self._ck(self._L.otdr_batch_get_plans(self._h, nat.dptr(X), nat.dptr(phi), nat.dptr(psi)))
        return X, phi, psi

    def states(self, with_plan: bool = True) -> list:
        """Each problem's complete final SolverState (solver.hpp:51-59)."""
        B, m, n = self.batch, self.m, self.n
        X = np.empty((B, m, n)) if with_plan else None
        rows = [np.empty((B, m)) for _ in range(3)]   # phi, a, r
        cols = [np.empty((B, n)) for _ in range(3)]   # psi, b, s
        theta, eta = np.empty(B), np.empty(B)
        k = np.empty(B, dtype=np.int64)
        self._ck(self._L.otdr_batch_get_state(
            self._h, nat.dptr(X) if X is not None else None, nat.dptr(rows[0]), nat.dptr(cols[0]),
            nat.dptr(rows[1]), nat.dptr(cols[1]), nat.dptr(rows[2]), nat.dptr(cols[2]),
            nat.dptr(theta), nat.dptr(eta), k.ctypes.data_as(ct.POINTER(ct.c_int64))))
        return [SolverState(X[b] if X is not None else None, rows[0][b], cols[0][b], rows[1][b],
                            cols[1][b], float(theta[b]), rows[2][b], cols[2][b], float(eta[b]),
                            int(k[b])) for b in range(B)]


def solve_batch(problems, reg: Regularizer, options: Optional[SolverOptions] = None) -> list:
    """`[solve(pr, reg, options) for pr in problems]` for same-shape problems,
    in one device launch; shapes beyond a cluster fall back to per-problem
    device solves (still on the GPU)."""
    opt = options or SolverOptions()
    if not problems:
        return []
    if opt.init is not None or opt.tol_gap is not None or opt.record_trace or opt.fused:
        return [solve(pr, reg, opt) for pr in problems]
    m, n = problems[0].rows(), problems[0].cols()
    if any(pr.cost.shape != (m, n) for pr in problems):
        raise DimensionMismatch("solve_batch needs problems of one shape")
    try:
        be = BatchEngine(len(problems), m, n, opt.storage, opt.device)
    except Unsupported:
        return [solve(pr, reg, opt) for pr in problems]
    be.set_problems(np.stack([pr.cost for pr in problems]), np.stack([pr.p for pr in problems]),
                    np.stack([pr.q for pr in problems]))
    be.set_regularizer(reg)
    reps = be.solve(opt)
    for rep, st in zip(reps, be.states()):
        rep.state = st  # the full final state, as solve() returns it (solver.hpp:74-87)
    be.close()
    return reps


def _engine_for(problem: Problem, storage: str, device: int) -> Engine:
    key = (storage, device)
    eng = problem._engines.get(key)
    if eng is None:
        eng = Engine(problem.rows(), problem.cols(), storage, device)
        eng.set_problem(problem.cost, problem.p, problem.q)
        problem._engines[key] = eng
    return eng


def make_state(problem: Problem, init: Optional[WarmStart] = None, storage: str = "f64",
               device: int = 0) -> SolverState:
    """solver.cpp:68-93 (seeding runs on device)."""
    eng = _engine_for(problem, storage, device)
    eng.set_regularizer(ZeroReg())
    eng.set_state(init)
    return eng.get_state()


def step(state: SolverState, problem: Problem, reg: Regularizer, rho: float,
         storage: str = "f64", device: int = 0) -> None:
    """One full DR iteration in place (solver.cpp:95-102)."""
    eng = _engine_for(problem, storage, device)
    eng.set_regularizer(reg)
    eng.load_state(state)
    eng.step(rho, 1)
    new = eng.get_state()
    state.X[...] = new.X
    for name in ("phi", "psi", "a", "b", "r", "s"):
        getattr(state, name)[...] = getattr(new, name)
    state.theta, state.eta, state.k = new.theta, new.eta, new.k


def solve(problem: Problem, reg: Regularizer, options: Optional[SolverOptions] = None) -> SolveReport:
    """solver.cpp:104-241, device-resident loop. Raises the reference's errors."""
    opt = options or SolverOptions()
    if opt.max_iter <= 0:
        raise ZeroIterations(f"max_iter must be positive, got {opt.max_iter}")
    if opt.check_every <= 0:
        raise InvalidArgument("check_every must be positive")
    if not (opt.tol_primal > 0.0):
        raise InvalidArgument("tol_primal must be positive")
    if opt.tol_gap is not None and not (opt.tol_gap > 0.0):
        raise InvalidArgument("tol_gap must be positive when set")
    eng = _engine_for(problem, opt.storage, opt.device)
    eng.set_regularizer(reg)
    eng.set_state(opt.init)
    return eng.solve(opt)


def primal_objective(problem: Problem, plan, reg: Regularizer, storage: str = "f64",
                     device: int = 0) -> float:
    """<C,X> + h(X) (problem.cpp:76-85), evaluated by the device objective kernel."""
    plan = _f64(plan)
    if plan.shape != (problem.rows(), problem.cols()):
        raise DimensionMismatch(f"plan is {plan.shape[0]}x{plan.shape[1]}, problem is "
                                f"{problem.rows()}x{problem.cols()}")
    eng = _engine_for(problem, storage, device)
    eng.set_regularizer(reg)
    eng.set_state(WarmStart(plan, np.zeros(problem.rows()), np.zeros(problem.cols())))
    return eng.objective()


def recover_duals(state: SolverState, rho: float):  # duality.cpp:5-7
    return state.phi / rho, state.psi / rho


def duality_gap(problem: Problem, reg: Regularizer, state: SolverState, rho: float,
                storage: str = "f64", device: int = 0) -> DualCertificate:
    """duality.cpp:9-24 on device (one clamp pass + objective)."""
    eng = _engine_for(problem, storage, device)
    eng.set_regularizer(reg)
    eng.load_state(state)
    dv, gap, dres = eng.duality_gap(rho)
    mu, nu = recover_duals(state, rho)
    return DualCertificate(mu, nu, dv, gap, dres)


def ot_cost_gradient(problem: Problem, reg: Regularizer, options: Optional[SolverOptions] = None):
    """duality.cpp:26-31: (objective, plan) of a solve."""
    rep = solve(problem, reg, options)
    return rep.objective, rep.plan()


def compute_skip_count(problem: Problem, rho: float = 0.0) -> int:
    """solver.cpp:243-256 (diagnostics only; setup-time host computation)."""
    m, n = float(problem.rows()), float(problem.cols())
    denom = m * problem.p[:, None] + n * problem.q[None, :] + 1.0
    term = np.ceil(problem.cost * m * n / (m + n) / denom - 1.0)
    return max(0, int(term.min()))
