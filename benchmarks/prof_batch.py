import sys, os
sys.path.insert(0, os.getcwd())
import torch
import numpy as np
import paper_2305_18483_b200 as otdr
from paper_2305_18483_b200 import datagen
B, m = 32, 512
src = np.empty((B, m, 2)); tgt = np.empty((B, m, 2))
for b in range(B):
    src[b], tgt[b] = datagen.gaussian_points(m, m, b)
ps = np.full((B, m), 1.0 / m)
be = otdr.BatchEngine(B, m, m, "f32")
be.build_sqdist_costs(src, tgt, ps, ps)
be.set_regularizer(otdr.QuadraticReg(5.12))
reps = be.solve(otdr.SolverOptions(tol_primal=1e-4, max_iter=20000))
print(sum(r.iterations for r in reps), reps[0].device_ms)
