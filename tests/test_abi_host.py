"""CPU-side checks: the C-ABI library loads and exports every declared symbol,
fails loudly without a GPU, and the host-side mirror of the reference API
(validation, partitions, skip count) agrees with the oracle."""
import os
import re

import numpy as np
import pytest

import paper_2305_18483_b200 as otdr
from paper_2305_18483_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for hdr in ("otdr_dev.h", "otdr_datagen.h"):
        src = open(os.path.join(ROOT, "include", hdr)).read()
        names |= set(re.findall(r"^\S.*\b(otdr_\w+)\s*\(", src, flags=re.M))
    return sorted(names)


def test_library_exports_every_declared_symbol():
    L = _native.lib()
    decl = declared_symbols()
    assert len(decl) >= 15
    for name in decl:
        assert hasattr(L, name), name
    assert sorted(_native.EXPORTS) == decl
    assert L.otdr_dev_abi_version() == 1


def test_no_cpu_fallback_without_gpu():
    L = _native.lib()
    if L.otdr_dev_cuda_available():
        pytest.skip("a CUDA device is present")
    with pytest.raises(otdr.DeviceError):
        otdr.Engine(4, 4)
    pr = otdr.validate_problem([[0, 1], [1, 0]], [0.5, 0.5], [0.5, 0.5])
    with pytest.raises(otdr.DeviceError):
        otdr.solve(pr, otdr.ZeroReg())


def test_validate_problem_mirrors_oracle(ora):
    rng = ora.Rng(7)
    for _ in range(20):
        C = np.array([[rng.uniform01() for _ in range(4)] for _ in range(3)])
        p = np.array([rng.uniform01() + 0.05 for _ in range(3)])
        q = np.array([rng.uniform01() + 0.05 for _ in range(4)])
        p = p * ((1 + 3e-7) / p.sum())
        q = q * ((1 - 3e-7) / q.sum())
        a = otdr.validate_problem(C, p, q)
        b = ora.validate_problem(C, p, q)
        assert np.allclose(a.p, b[1], rtol=0, atol=1e-16) and np.allclose(a.q, b[2], rtol=0, atol=1e-16)
        again = otdr.validate_problem(a.cost, a.p, a.q)
        assert np.array_equal(again.p, a.p) and np.array_equal(again.q, a.q)
    c = [[0, 1], [1, 0]]
    with pytest.raises(otdr.MarginalSumOutOfRange):
        otdr.validate_problem(c, [0.5, 0.6], [0.5, 0.5])
    with pytest.raises(otdr.NegativeEntry):
        otdr.validate_problem([[-1, 0], [0, 1]], [0.5, 0.5], [0.5, 0.5])
    with pytest.raises(otdr.NegativeEntry):
        otdr.validate_problem(c, [np.nan, 1], [0.5, 0.5])
    with pytest.raises(otdr.DimensionMismatch):
        otdr.validate_problem(c, [1 / 3] * 3, [0.5, 0.5])
    with pytest.raises(otdr.DimensionMismatch):
        otdr.validate_problem(np.zeros((0, 0)), [], [])
    n, z = otdr.normalize_cost(otdr.validate_problem([[2, 4], [1, 3]], [0.5, 0.5], [0.5, 0.5]), True)
    assert np.array_equal(n.cost, [[0.5, 1.0], [0.25, 0.75]]) and not z


def test_column_class_blocks_matches_oracle(ora):
    for labels, n in (([0, 0, 0, 0], 3), ([0, 1, 0, 1], 3), ([1, 0, 2, 1, 0], 4), ([0, 0, 3, 3], 2)):
        part = otdr.column_class_blocks(labels, n)
        offs, cells = ora.column_class_blocks(labels, n)
        assert np.array_equal(part.offsets, offs) and np.array_equal(part.cells, cells)
        # a generic partition with the same groups recovers the same row classes
        groups = [[tuple(c) for c in cells[offs[g]:offs[g + 1]]] for g in range(len(offs) - 1)]
        generic = otdr.make_partition(len(labels), n, groups)
        lab = otdr.otdr._labels_of(generic)
        for i in range(len(labels)):
            for k in range(len(labels)):
                assert (lab[i] == lab[k]) == (labels[i] == labels[k])
    with pytest.raises(otdr.InvalidArgument):
        otdr.column_class_blocks([0, -1], 2)
    with pytest.raises(otdr.InvalidArgument):
        otdr.make_partition(2, 2, [[(0, 0), (0, 1)], [(0, 1)]])
    # a group spanning two columns has no kernel: Unsupported, not a CPU fallback
    with pytest.raises(otdr.Unsupported):
        otdr.otdr._labels_of(otdr.make_partition(2, 2, [[(0, 0), (0, 1)]]))


def test_skip_count_and_init_mirror_oracle(ora):
    n = 100
    big = otdr.validate_problem(np.ones((n, n)), np.full(n, 1 / n), np.full(n, 1 / n))
    assert otdr.compute_skip_count(big) == 16
    w = otdr.default_init(2, 3)
    assert w.phi0[0] == pytest.approx(1.4 / 15, rel=1e-15) and w.psi0[0] == pytest.approx(1.6 / 15, rel=1e-15)
    assert otdr.default_stepsize(2000, 3000) == pytest.approx(4e-4, rel=1e-15)
    with pytest.raises(otdr.InvalidArgument):
        otdr.QuadraticReg(0.0)
    with pytest.raises(otdr.InvalidArgument):
        otdr.GroupLassoReg(-1.0, otdr.column_class_blocks([0], 1))


def test_otpb_host_roundtrip(tmp_path):
    from paper_2305_18483_b200 import io
    a = np.arange(12, dtype=np.float64).reshape(3, 4) / 7.0
    path = str(tmp_path / "a.otpb")
    io.write_matrix_otpb(path, a)
    raw = open(path, "rb").read()
    assert raw[:4] == b"OTPB" and raw[4:8] == (3).to_bytes(4, "little") and raw[12:16] == b"\0" * 4
    assert len(raw) == 16 + 12 * 8
    assert np.array_equal(io.read_matrix_otpb(path), a)
    open(path, "r+b").write(b"XXXX")
    with pytest.raises(otdr.InvalidArgument):
        io.read_matrix_otpb(path)


def test_sass_memory_descriptors_are_even_register_pairs():
    """Every global access in the built kernels addresses its 64-bit memory
    descriptor through an even uniform-register pair. ptxas 12.9 once emitted
    desc[UR1] for a cp.async with an L2 cache-policy operand, which faults as
    an illegal instruction on B200; this guards the build against that."""
    import re
    import shutil
    import subprocess

    lib = os.path.join(ROOT, "paper_2305_18483_b200", "libotdr_dev.so")
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(lib) or not os.path.exists(tool):
        pytest.skip("library or cuobjdump missing")
    sass = subprocess.run([tool, "-sass", lib], capture_output=True, text=True).stdout
    regs = {int(r) for r in re.findall(r"desc\[UR(\d+)\]", sass)}
    assert regs, "no SASS found"
    assert all(r % 2 == 0 for r in regs), sorted(regs)
