"""World-size-2 gloo tests of the row-sharded decomposition (CPU).

The device path shards the plan by rows and all-reduces [S | sum r | sum r^2 |
sum X] once per iteration (paper_2305_18483_b200/sharding.py, update_kernel).
Here two CPU processes run exactly that decomposition over the oracle's
row-local sweep with a gloo all-reduce, and must reproduce the unsharded
oracle trajectory; the band planner and NCCL-id broadcast are exercised too.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sharded_worker(rank, world, port, kind, out):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    import torch

    import pyoracle as ora
    from paper_2305_18483_b200 import sharding

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, n = 23, 17
        C, p, q, *_ = ora.adaptation_problem(m, n, 3, 4)
        _, _, _, _, _, labels, _ = ora.adaptation_problem(m, n, 3, 4)
        bands = sharding.row_bands(m, world, labels if kind == "gl" else None)
        lo, hi = bands[rank]
        rho = ora.default_stepsize(m, n)
        if kind == "quad":
            reg = ora.quad_reg(3.0)
        elif kind == "gl":
            offs, cells = ora.column_class_blocks(labels[lo:hi], n)
            reg = ora.group_lasso_reg(0.01, offs, cells)
        else:
            reg = ora.zero_reg()
        # make_state on the band (solver.cpp:68-93), global sums all-reduced
        X = np.zeros((hi - lo, n))
        mn = float(m + n)
        phi = np.full(hi - lo, (1.0 + m / mn) / (3.0 * mn))
        psi = np.full(n, (1.0 + n / mn) / (3.0 * mn))

        def exchange(Xb):
            R = Xb.sum(axis=1)
            r = R - p[lo:hi]
            buf = torch.tensor(np.concatenate([Xb.sum(axis=0), [r.sum(), (r * r).sum(), R.sum()]]),
                               dtype=torch.float64)
            dist.all_reduce(buf)
            return r, buf.numpy()

        r, ex = exchange(X)
        s = ex[:n] - q
        a = n * phi + r
        b = m * psi + s
        theta = (ex[n + 2] - 1.0) / (m + n)
        for _ in range(30):
            V = np.maximum(((X - rho * C[lo:hi]) + phi[:, None]) + psi[None, :], 0.0)
            X = ora.prox(reg, V, rho)
            r, ex = exchange(X)
            s = ex[:n] - q
            eta = ex[n] / (m + n)
            shift = 2.0 * eta - theta
            phi = ((a - 2.0 * r) + shift) / n
            psi = ((b - 2.0 * s) + shift) / m
            a = a - r
            b = b - s
            theta -= eta
        Xall = [None] * world
        dist.all_gather_object(Xall, (lo, hi, X, phi, psi))
        if rank == 0:
            out.put((bands, Xall))
        if kind == "none":
            nid = sharding.broadcast_nccl_id(dist, rank)
            got = [None] * world
            dist.all_gather_object(got, nid)
            assert len(nid) == 128 and got[0] == got[1]
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["none", "quad", "gl"])
def test_row_sharded_recurrence_matches_unsharded(ora, kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    bands, parts = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    m, n = 23, 17
    C, p, qq, *_ = ora.adaptation_problem(m, n, 3, 4)
    labels = ora.adaptation_problem(m, n, 3, 4)[5]
    pr_ = ora.Problem(C, p, qq)
    if kind == "quad":
        reg = ora.quad_reg(3.0)
    elif kind == "gl":
        reg = ora.group_lasso_reg(0.01, *ora.column_class_blocks(labels, n))
    else:
        reg = ora.zero_reg()
    st = ora.make_state(pr_)
    for _ in range(30):
        ora.step(st, pr_, reg, ora.default_stepsize(m, n))
    X = np.vstack([x for (_, _, x, _, _) in parts])
    phi = np.concatenate([ph for (_, _, _, ph, _) in parts])
    assert bands[0][0] == 0 and bands[-1][1] == m and bands[0][1] == bands[1][0]
    scale = np.abs(st.X).max()
    assert np.abs(X - st.X).max() <= 1e-12 * scale
    assert np.abs(phi - st.phi).max() <= 1e-12 * np.abs(st.phi).max()
    assert np.abs(parts[0][4] - st.psi).max() <= 1e-12 * np.abs(st.psi).max()
    assert np.array_equal(parts[0][4], parts[1][4])  # replicated psi identical on all ranks


def test_row_bands_class_alignment():
    from paper_2305_18483_b200 import Unsupported, sharding

    assert sharding.row_bands(10, 3) == [(0, 3), (3, 6), (6, 10)]
    lab = [0] * 7 + [1] * 2 + [2] * 11
    bands = sharding.row_bands(20, 2, lab)
    assert bands == [(0, 9), (9, 20)]
    for lo, hi in sharding.row_bands(20, 4, lab):
        assert lo == hi or len(set(lab[lo:hi])) >= 1
    cuts = {b for (_, b) in sharding.row_bands(20, 4, lab)}
    assert cuts <= {0, 7, 9, 20}
    with pytest.raises(Unsupported):
        sharding.row_bands(4, 2, [0, 1, 0, 1])  # interleaved classes cannot be banded
    # ungrouped rows may be cut anywhere
    assert sharding.row_bands(6, 2, [-1] * 6) == [(0, 3), (3, 6)]
