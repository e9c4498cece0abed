"""OTPB matrix files (io.cpp:127-158 of the reference): 16-byte header
("OTPB", u32 m, u32 n, 4 zero bytes) then m*n fp64 row-major. Host helpers for
callers; the device engine reads costs into and writes plans out of HBM
directly (Engine.read_cost_otpb / Engine.write_plan_otpb)."""
from __future__ import annotations

import struct

import numpy as np

from .otdr import DimensionMismatch, InvalidArgument

MAGIC = b"OTPB"


def write_matrix_otpb(path: str, m: np.ndarray) -> None:
    a = np.ascontiguousarray(np.asarray(m, dtype="<f8"))
    if a.ndim != 2 or a.shape[0] < 1 or a.shape[1] < 1:
        raise DimensionMismatch("OTPB needs a non-empty 2-D matrix")
    with open(path, "wb") as f:
        f.write(MAGIC + struct.pack("<II", a.shape[0], a.shape[1]) + b"\0" * 4)
        f.write(a.tobytes())


def read_matrix_otpb(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        hdr = f.read(16)
        if len(hdr) != 16 or hdr[:4] != MAGIC:
            raise InvalidArgument(f"{path}: not an OTPB file (bad magic)")
        m, n = struct.unpack("<II", hdr[4:12])
        if m == 0 or n == 0:
            raise InvalidArgument(f"{path}: zero dimension in OTPB header")
        data = np.fromfile(f, dtype="<f8", count=m * n)
    if data.size != m * n:
        raise InvalidArgument(f"{path}: truncated OTPB payload")
    return data.reshape(m, n).astype(np.float64)
