#!/usr/bin/env python
"""cfg1 (1000^2 quadratic, alpha = 10) on the on-chip resident kernel: time
per iteration of a 2000-iteration launch, fp32 and fp64 storage (one JSON
line each). Used under ncu to profile the resident kernel:
  ncu --set full -k regex:resident -c 1 python benchmarks/cfg1_resident.py f32
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2305_18483_b200 as otdr  # noqa: E402
from paper_2305_18483_b200 import datagen  # noqa: E402

m = n = 1000
src, tgt = datagen.gaussian_points(m, n, 0)
for storage in sys.argv[1:] or ("f32", "f64"):
    eng = otdr.Engine(m, n, storage)
    eng.build_sqdist_cost(src, tgt, datagen.uniform(m), datagen.uniform(n))
    eng.set_regularizer(otdr.QuadraticReg(10.0))
    eng.set_state()
    rho = otdr.default_stepsize(m, n)
    eng.step(rho, 10)
    it = 2000
    ms = eng.time_steps(rho, it)
    print(json.dumps({"storage": storage, "kernel": eng.kernel_name(), "us_per_iter": 1e3 * ms / it}), flush=True)
    eng.close()
