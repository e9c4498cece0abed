#!/usr/bin/env python
"""Compare sweep-kernel variants (selected by environment variables, read at
Engine creation) on one config; one JSON line per variant.

  python benchmarks/variants.py headline OTDR_STREAM_KERNEL=tma OTDR_STREAM_KERNEL=async
  python benchmarks/variants.py cfg3 OTDR_GL_KERNEL=pipe OTDR_GL_KERNEL=twopass
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, os, sys
sys.path.insert(0, ROOT)
import torch
import paper_2305_18483_b200 as otdr
from paper_2305_18483_b200 import datagen
cfg = CFG
if cfg in ("headline", "cfg2", "cfg4", "cfg1") or cfg.startswith("n"):
    m = {"headline": 20000, "cfg2": 10000, "cfg4": 40000, "cfg1": 1000}.get(cfg) or int(cfg[1:].split("x")[0])
    nn = int(cfg[1:].split("x")[1]) if cfg.startswith("n") and "x" in cfg else m
    alpha = 5e-3 * 2 * m * float(os.environ.get("OTDRB_ALPHA_SCALE", "1"))
    reg = {"cfg2": otdr.ZeroReg()}.get(cfg, otdr.QuadraticReg(alpha))
    st = os.environ.get("OTDRB_STORAGE", "f32")
    eng = otdr.Engine(m, nn, st)
    src, tgt = datagen.gaussian_points(m, nn, 0)
    eng.build_sqdist_cost(src, tgt, datagen.uniform(m), datagen.uniform(nn))
else:
    m = 10000
    src, tgt, ls, lt = datagen.adaptation_points(m, m, 10, 0)
    eng = otdr.Engine(m, m, "f32")
    eng.build_sqdist_cost(src, tgt, datagen.uniform(m), datagen.uniform(m))
    reg = otdr.GroupLassoReg(1e-3, otdr.column_class_blocks(ls, m))
eng.set_regularizer(reg)
eng.set_state()
nn = locals().get("nn", m)
rho = otdr.default_stepsize(m, nn)
eng.step(rho, int(os.environ.get("OTDRB_PRESTEPS", "5")))
ms = eng.time_steps(rho, ITERS) / ITERS
prof = eng.profile(rho, 5)
alg = (24.0 if os.environ.get("OTDRB_STORAGE") == "f64" else 12.0) * m * nn
print("RESULT " + json.dumps(dict(cfg=cfg, variant=VARIANT, path=eng.solve_path(), ms_per_iter=ms, iters_per_s=1e3 / ms,
      nnz=float((eng.get_state().X[: min(m, 2000)] != 0).mean()) if os.environ.get("OTDRB_NNZ") else None,
      sweep_ms=prof["sweep_ms"], sweep_GBps=alg / prof["sweep_ms"] / 1e6,
      iter_GBps=alg / ms / 1e6, prof=prof)), flush=True)
"""


def main():
    cfg = sys.argv[1]
    iters = {"cfg4": 30, "cfg1": 2000}.get(cfg, 100 if not cfg.startswith("n") else
                                          max(30, min(2000, int(4e10 / eval(cfg[1:].replace("x", "*")) / (1 if "x" in cfg else int(cfg[1:]))))))
    for var in sys.argv[2:] or ["default"]:
        env = dict(os.environ)
        for kv in var.split(","):
            if "=" in kv:
                k, v = kv.split("=", 1)
                env[k] = v
        code = CHILD.replace("ROOT", repr(ROOT)).replace("CFG", repr(cfg)) \
                    .replace("ITERS", str(iters)).replace("VARIANT", repr(var))
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        got = [l[7:] for l in out.stdout.splitlines() if l.startswith("RESULT ")]
        if got:
            print(got[0], flush=True)
        else:
            print(json.dumps(dict(cfg=cfg, variant=var, error=(out.stderr or out.stdout)[-800:])), flush=True)


if __name__ == "__main__":
    main()
