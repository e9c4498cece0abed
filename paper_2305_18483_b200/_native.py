"""ctypes binding of libotdr_dev.so (the C-ABI in include/otdr_dev.h).

The library is built in-tree (paper_2305_18483_b200/libotdr_dev.so, see
csrc/Makefile). There is no CPU fallback: if the library is missing the import
of any solver entry point raises, and without a CUDA device every call that
needs one returns OTDR_E_CUDA.
"""
from __future__ import annotations

import ctypes as ct
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libotdr_dev.so")

OTDR_OK = 0
STATUS_NAMES = {
    0: "OK", 1: "DIMENSION", 2: "NEGATIVE", 3: "MARGINAL", 4: "ZERO_ITERS", 5: "INVALID_ARG",
    6: "NONFINITE", 7: "UNSUPPORTED", 8: "CUDA", 9: "NCCL", 10: "STATE",
}
REG_NONE, REG_QUAD, REG_GROUP_LASSO = 0, 1, 2
STORE_F32, STORE_F64 = 0, 1

_dp = ct.POINTER(ct.c_double)
_i32p = ct.POINTER(ct.c_int32)
_i64p = ct.POINTER(ct.c_int64)


class DevConfig(ct.Structure):
    _fields_ = [("device", ct.c_int), ("storage", ct.c_int), ("m", ct.c_int64), ("n", ct.c_int64),
                ("rank", ct.c_int), ("nranks", ct.c_int), ("row_begin", ct.c_int64),
                ("row_end", ct.c_int64), ("nccl_id", ct.c_char_p)]


class SolveOpts(ct.Structure):
    _fields_ = [("rho", ct.c_double), ("max_iter", ct.c_int64), ("tol_primal", ct.c_double),
                ("has_tol_gap", ct.c_int), ("tol_gap", ct.c_double), ("check_every", ct.c_int64),
                ("deterministic", ct.c_int), ("record_trace", ct.c_int), ("fused", ct.c_int)]


class SolveResult(ct.Structure):
    _fields_ = [("iterations", ct.c_int64), ("termination", ct.c_int), ("rho", ct.c_double),
                ("r_primal", ct.c_double), ("objective", ct.c_double),
                ("support_last_change", ct.c_int64), ("trace_rows", ct.c_int64),
                ("device_ms", ct.c_double)]


class TraceRow(ct.Structure):
    _fields_ = [("iter", ct.c_int64), ("r_primal", ct.c_double), ("gap", ct.c_double),
                ("dual_residual", ct.c_double), ("support", ct.c_int64), ("elapsed_ms", ct.c_double)]


class Certificate(ct.Structure):
    _fields_ = [("dual_value", ct.c_double), ("gap", ct.c_double), ("dual_residual", ct.c_double)]


class KernelTimes(ct.Structure):
    _fields_ = [("sweep_ms", ct.c_double), ("reduce_ms", ct.c_double), ("exchange_ms", ct.c_double),
                ("update_ms", ct.c_double), ("iterations", ct.c_int64), ("sweep_bytes", ct.c_double)]


PEER_HANDLE_BYTES = 64  # OTDR_PEER_HANDLE_BYTES

# Every symbol include/otdr_dev.h declares (checked by the CPU ABI test).
EXPORTS = [
    "otdr_dev_abi_version", "otdr_dev_create", "otdr_dev_destroy", "otdr_dev_last_error",
    "otdr_dev_cuda_available", "otdr_dev_set_problem", "otdr_dev_build_sqdist_cost",
    "otdr_dev_set_regularizer", "otdr_dev_set_state", "otdr_dev_load_state", "otdr_dev_step",
    "otdr_dev_solve", "otdr_dev_get_state", "otdr_dev_objective", "otdr_dev_duality_gap",
    "otdr_dev_get_trace", "otdr_dev_profile", "otdr_dev_time_steps",
    "otdr_dev_kernels_per_iteration", "otdr_dev_solve_path", "otdr_dev_kernel_name", "otdr_dev_peer_export",
    "otdr_dev_peer_import", "otdr_dev_peer_link_local", "otdr_dev_read_cost_otpb", "otdr_dev_write_plan_otpb",
    "otdr_batch_create", "otdr_batch_destroy", "otdr_batch_last_error", "otdr_batch_set_problems",
    "otdr_batch_build_sqdist_costs", "otdr_batch_set_regularizer", "otdr_batch_solve",
    "otdr_batch_get_plans", "otdr_batch_get_state",
    # include/otdr_datagen.h
    "otdr_gaussian_points", "otdr_adaptation_points", "otdr_dev_nccl_unique_id",
]

_lib = None


def lib():
    """Load libotdr_dev.so (raises loudly when it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C paper_2305_18483_b200/csrc` "
            "(there is no CPU fallback)")
    L = ct.CDLL(LIB_PATH)
    vp = ct.c_void_p
    L.otdr_dev_abi_version.restype = ct.c_int
    L.otdr_dev_cuda_available.restype = ct.c_int
    L.otdr_dev_create.argtypes = [ct.POINTER(DevConfig), ct.POINTER(vp)]
    L.otdr_dev_destroy.argtypes = [vp]
    L.otdr_dev_destroy.restype = None
    L.otdr_dev_last_error.argtypes = [vp]
    L.otdr_dev_last_error.restype = ct.c_char_p
    L.otdr_dev_set_problem.argtypes = [vp, _dp, _dp, _dp]
    L.otdr_dev_build_sqdist_cost.argtypes = [vp, _dp, _dp, ct.c_int, _dp, _dp, ct.POINTER(ct.c_int)]
    L.otdr_dev_set_regularizer.argtypes = [vp, ct.c_int, ct.c_double, _i32p]
    L.otdr_dev_set_state.argtypes = [vp, _dp, _dp, _dp]
    L.otdr_dev_load_state.argtypes = [vp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, ct.c_double,
                                      ct.c_double, ct.c_int64]
    L.otdr_dev_step.argtypes = [vp, ct.c_double, ct.c_int64]
    L.otdr_dev_solve.argtypes = [vp, ct.POINTER(SolveOpts), ct.POINTER(SolveResult)]
    L.otdr_dev_get_state.argtypes = [vp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _i64p]
    L.otdr_dev_objective.argtypes = [vp, _dp]
    L.otdr_dev_duality_gap.argtypes = [vp, ct.c_double, ct.POINTER(Certificate)]
    L.otdr_dev_get_trace.argtypes = [vp, ct.POINTER(TraceRow), ct.c_int64, _i64p]
    L.otdr_dev_profile.argtypes = [vp, ct.c_double, ct.c_int64, ct.POINTER(KernelTimes)]
    L.otdr_dev_time_steps.argtypes = [vp, ct.c_double, ct.c_int64, _dp]
    L.otdr_dev_read_cost_otpb.argtypes = [vp, ct.c_char_p, _dp, _dp]
    L.otdr_dev_write_plan_otpb.argtypes = [vp, ct.c_char_p]
    L.otdr_gaussian_points.argtypes = [ct.c_int64, ct.c_int64, ct.c_uint64, _dp, _dp]
    L.otdr_gaussian_points.restype = None
    L.otdr_adaptation_points.argtypes = [ct.c_int64, ct.c_int64, ct.c_int, ct.c_uint64, ct.c_int,
                                         _dp, _dp, _i32p, _i32p]
    L.otdr_dev_nccl_unique_id.argtypes = [ct.c_char_p]
    L.otdr_batch_create.argtypes = [ct.c_int, ct.c_int, ct.c_int64, ct.c_int64, ct.c_int64,
                                    ct.POINTER(vp)]
    L.otdr_batch_destroy.argtypes = [vp]
    L.otdr_batch_destroy.restype = None
    L.otdr_batch_last_error.argtypes = [vp]
    L.otdr_batch_last_error.restype = ct.c_char_p
    L.otdr_batch_set_problems.argtypes = [vp, _dp, _dp, _dp]
    L.otdr_batch_build_sqdist_costs.argtypes = [vp, _dp, _dp, ct.c_int, _dp, _dp]
    L.otdr_batch_set_regularizer.argtypes = [vp, ct.c_int, ct.c_double]
    L.otdr_batch_solve.argtypes = [vp, ct.POINTER(SolveOpts), ct.POINTER(SolveResult)]
    L.otdr_batch_get_plans.argtypes = [vp, _dp, _dp, _dp]
    L.otdr_batch_get_state.argtypes = [vp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                       ct.POINTER(ct.c_int64)]
    L.otdr_dev_kernels_per_iteration.argtypes = [vp]
    L.otdr_dev_kernels_per_iteration.restype = ct.c_int
    L.otdr_dev_solve_path.argtypes = [vp]
    L.otdr_dev_solve_path.restype = ct.c_int
    L.otdr_dev_kernel_name.argtypes = [vp]
    L.otdr_dev_kernel_name.restype = ct.c_char_p
    L.otdr_dev_peer_export.argtypes = [vp, ct.c_char_p]
    L.otdr_dev_peer_export.restype = ct.c_int
    L.otdr_dev_peer_import.argtypes = [vp, ct.c_char_p]
    L.otdr_dev_peer_import.restype = ct.c_int
    L.otdr_dev_peer_link_local.argtypes = [ct.POINTER(vp), ct.c_int]
    L.otdr_dev_peer_link_local.restype = ct.c_int
    _lib = L
    return L


def dptr(a):
    return None if a is None else a.ctypes.data_as(_dp)
