"""Worker of test_peer_ipc_two_processes (launched by torch.distributed.run):
two processes = two ranks of a row-sharded run on ONE GPU, exchanging over
CUDA IPC peer memory (handles all-gathered with gloo). Rank 0 checks the
gathered iterates against the unsharded oracle and prints PEER_IPC_OK."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2305_18483_b200 as otdr  # noqa: E402
from paper_2305_18483_b200 import sharding  # noqa: E402
import pyoracle as ora  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    m, n, k = 600, 500, 12
    C, p, q, *_ = ora.gaussian_problem(m, n, 7)
    lo, hi = sharding.row_bands(m, world)[rank]
    eng = otdr.Engine(m, n, "f64", device=0, shard=otdr.Shard(rank, world, lo, hi, None))
    eng.set_problem(C[lo:hi], p[lo:hi], q)
    eng.set_regularizer(otdr.QuadraticReg(0.8))
    sharding.connect_peers(dist, eng)
    eng.set_state()
    rho = otdr.default_stepsize(m, n)
    eng.step(rho, k)
    g = eng.get_state()
    parts = [None] * world
    dist.all_gather_object(parts, (g.X, g.phi, g.psi, g.k))
    if rank == 0:
        pr = ora.Problem(C, p, q)
        st = ora.make_state(pr)
        for _ in range(k):
            ora.step(st, pr, ora.quad_reg(0.8), rho)
        X = np.concatenate([x for x, _, _, _ in parts])
        phi = np.concatenate([f for _, f, _, _ in parts])
        err = float(np.abs(X - st.X).max() / np.abs(st.X).max())
        errp = float(np.abs(phi - st.phi).max() / np.abs(st.phi).max())
        errs = max(float(np.abs(ps - st.psi).max() / np.abs(st.psi).max()) for _, _, ps, _ in parts)
        assert all(kk == k for *_, kk in parts)
        assert err <= 1e-12 and errp <= 1e-12 and errs <= 1e-12, (err, errp, errs)
        print("PEER_IPC_OK", err, flush=True)
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
