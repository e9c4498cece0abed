"""Where the bench's end-to-end step goes: H2D cost upload, make_state, device
solve (the reference's default options: tol 1e-4), D2H plan download -- host
wall clock, 20000^2 fp32 storage, host buffers in ordinary pageable memory (as
bench.py's e2e) or pinned (--pinned). OTDR_HOST_THREADS sets the conversion
threads of the upload / download pipeline."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2305_18483_b200 as otdr  # noqa: E402
from paper_2305_18483_b200 import datagen  # noqa: E402

M = N = 20000
pinned = "--pinned" in sys.argv
src, tgt = datagen.gaussian_points(M, N, 0)
alloc = (lambda: torch.empty((M, N), dtype=torch.float64, pin_memory=True).numpy()) if pinned \
    else (lambda: np.empty((M, N)))
C = alloc()
for r0 in range(0, M, 2000):
    C[r0:r0 + 2000] = datagen.squared_distance_cost(src[r0:r0 + 2000], tgt)
C /= C.max()
p, q = datagen.uniform(M), datagen.uniform(N)
plan = alloc()
plan.fill(0.0)
eng = otdr.Engine(M, N, "f32")
opts = otdr.SolverOptions(storage="f32")
for rep in range(3):
    t = [time.perf_counter()]
    eng.set_problem(C, p, q); t.append(time.perf_counter())
    eng.set_regularizer(otdr.QuadraticReg(200.0)); eng.set_state(); t.append(time.perf_counter())
    r = eng.solve(opts, with_state=False); t.append(time.perf_counter())
    eng.get_plan_into(plan); t.append(time.perf_counter())
    d = [b - a for a, b in zip(t, t[1:])]
    print(json.dumps({"rep": rep, "pinned": pinned, "threads": os.environ.get("OTDR_HOST_THREADS", "default"),
                      "upload_s": d[0], "state_s": d[1], "solve_s": d[2], "download_s": d[3],
                      "total_s": t[-1] - t[0], "iterations": r.iterations, "device_ms": r.device_ms,
                      "h2d_GBps_fp64": 3.2 / d[0], "d2h_GBps_fp64": 3.2 / d[3]}), flush=True)
