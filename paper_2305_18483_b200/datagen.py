"""Seeded benchmark instances (datagen.cpp:21-129 restated in
csrc/otdr_datagen.cpp; the cost is built on device or in numpy below)."""
from __future__ import annotations

import ctypes as ct

import numpy as np

from . import _native as nat
from .otdr import InvalidArgument, Problem, column_class_blocks, normalize_cost, validate_problem


def gaussian_points(m: int, n: int, seed: int):
    """The two 2-D Gaussian clouds of gaussian_problem(m, n, seed)."""
    src = np.empty((m, 2))
    tgt = np.empty((n, 2))
    nat.lib().otdr_gaussian_points(m, n, seed, nat.dptr(src), nat.dptr(tgt))
    return src, tgt


def adaptation_points(m: int, n: int, classes: int, seed: int, identity_map: bool = False):
    src = np.empty((m, 2))
    tgt = np.empty((n, 2))
    ls = np.empty(m, dtype=np.int32)
    lt = np.empty(n, dtype=np.int32)
    i32 = ct.POINTER(ct.c_int32)
    rc = nat.lib().otdr_adaptation_points(m, n, classes, seed, int(identity_map), nat.dptr(src),
                                          nat.dptr(tgt), ls.ctypes.data_as(i32),
                                          lt.ctypes.data_as(i32))
    if rc:
        raise InvalidArgument("adaptation_problem: need classes >= 1 and a point per class")
    return src, tgt, ls, lt


def squared_distance_cost(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """C_ij = 0.5 ||a_i - b_j||^2 (datagen.cpp:43-54), host fp64 (d = 2 order)."""
    d0 = a[:, 0:1] - b[None, :, 0]
    d1 = a[:, 1:2] - b[None, :, 1]
    return 0.5 * (d0 * d0 + d1 * d1)


def uniform(n: int) -> np.ndarray:
    return np.full(n, 1.0 / n)


def gaussian_problem(m: int, n: int, seed: int):
    """(Problem, source, target) as datagen.cpp:56-65 builds them (host cost)."""
    src, tgt = gaussian_points(m, n, seed)
    pr = normalize_cost(validate_problem(squared_distance_cost(src, tgt), uniform(m), uniform(n)))
    return pr, src, tgt


def adaptation_problem(m: int, n: int, classes: int, seed: int, identity_map: bool = False):
    """(Problem, groups, src, tgt, src_labels, tgt_labels) as datagen.cpp:67-129."""
    src, tgt, ls, lt = adaptation_points(m, n, classes, seed, identity_map)
    pr = normalize_cost(validate_problem(squared_distance_cost(src, tgt), uniform(m), uniform(n)))
    return pr, column_class_blocks(ls, n), src, tgt, ls, lt
