#!/usr/bin/env python
"""Per-rank iteration time of a row-sharded run, measured on ONE GPU.

Rank r of an N-GPU run of the headline problem (20000 x 20000) sweeps a
(20000 / N) x 20000 band and exchanges the n+3 vector. On one GPU we time that
band with the peer-exchange streaming kernel linked to itself (1-rank peer
group: the flag publish / wait and the rank-order fold run, only the NVLink
hop is missing) and without the exchange, and print one JSON line per N.
OTDRB_M=40000 projects config 4 (40000 x 40000 quadratic, alpha = 5e-3 (m+n)).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: F401,E402

import paper_2305_18483_b200 as otdr  # noqa: E402
from paper_2305_18483_b200 import datagen  # noqa: E402

M = N = int(os.environ.get("OTDRB_M", "20000"))
src, tgt = datagen.gaussian_points(M, N, 0)
for world in [int(w) for w in sys.argv[1:]] or (1, 2, 4, 8):
    rows = M // world
    out = {"n_gpus_projected": world, "band_rows": rows, "n": N}
    for mode in ("plain", "peer1"):
        eng = otdr.Engine(rows, N, "f32")
        if mode == "peer1":  # 1-rank peer group over the band
            otdr.link_local([eng])
        eng.build_sqdist_cost(src[:rows], tgt, datagen.uniform(rows), datagen.uniform(N))
        eng.set_regularizer(otdr.QuadraticReg(5e-3 * (M + N)))
        eng.set_state()
        rho = otdr.default_stepsize(M, N)
        eng.step(rho, 5)
        it = 200
        ms = eng.time_steps(rho, it) / it
        out[mode + "_us_per_iter"] = ms * 1e3
        out[mode + "_path"] = eng.solve_path()
        out[mode + "_GBps"] = 12.0 * rows * N / (ms * 1e-3) / 1e9
        eng.close()
    print(json.dumps(out), flush=True)
