"""Plan sparsity along a 20000^2 quadratic solve: fraction of non-zero entries
and of all-zero 128-byte lines (what generic HBM compression can skip)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import paper_2305_18483_b200 as otdr
from paper_2305_18483_b200 import datagen
m = n = 20000
src, tgt = datagen.gaussian_points(m, n, 0)
eng = otdr.Engine(m, n, "f32")
eng.build_sqdist_cost(src, tgt, datagen.uniform(m), datagen.uniform(n))
eng.set_regularizer(otdr.QuadraticReg(200.0))
eng.set_state()
rho = otdr.default_stepsize(m, n)
done = 0
for k in (10, 100, 300, 1000):
    eng.step(rho, k - done); done = k
    X = eng.get_state().X.astype(np.float32)
    nz = float((X != 0).mean())
    lines = X[:, : (n // 32) * 32].reshape(m, -1, 32)
    zl = float((np.abs(lines).max(axis=2) == 0).mean())
    print(f"k={k} nonzero frac {nz:.4f} all-zero 128B lines {zl:.4f}", flush=True)
