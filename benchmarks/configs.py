#!/usr/bin/env python
"""Per-config measurements of the BASELINE.json configs (one JSON line each).

bench.py carries the driver's headline line (20000^2 quadratic); this script
measures the other configs on one GPU for DESIGN.md / profiles/:

  cfg1  quadratic 1000^2, alpha = 5e-3 (m+n), tol 1e-4     (L2-resident, latency-bound)
  cfg2  unregularized 10000^2 fp32                          (HBM-bound)
  cfg3  group lasso 10000^2, 10 class row groups, lambda 1e-3 / 0.06
  cfg4  quadratic 40000^2 on one GPU (the multi-GPU config's N=1 point)
  cfg5  batched 512^2 x 256 quadratic (sequential engine solves)

Usage: python benchmarks/configs.py [cfg1 cfg2 ...] [--fused] [--iters K]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
try:
    import torch  # noqa: F401  (load its NCCL before libotdr_dev.so)
except Exception:
    pass

import numpy as np  # noqa: E402

import paper_2305_18483_b200 as otdr  # noqa: E402
from paper_2305_18483_b200 import datagen  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def gaussian_engine(m, n, seed, storage="f32"):
    eng = otdr.Engine(m, n, storage)
    src, tgt = datagen.gaussian_points(m, n, seed)
    eng.build_sqdist_cost(src, tgt, datagen.uniform(m), datagen.uniform(n))
    return eng


def steady(eng, rho, iters):
    eng.step(rho, 5)
    ms = eng.time_steps(rho, iters)
    prof = eng.profile(rho, 5)
    return ms / iters, prof


def line(cfg, **kw):
    d = {"config": cfg}
    d.update(kw)
    print(json.dumps(d), flush=True)


def run_plain(cfg, m, n, reg, storage, iters, tol=1e-4, fused=False, max_iter=20000):
    eng = gaussian_engine(m, n, 0, storage)
    eng.set_regularizer(reg)
    eng.set_state()
    rho = otdr.default_stepsize(m, n)
    ms_it, prof = steady(eng, rho, iters)
    eng.set_state()
    rep = eng.solve(otdr.SolverOptions(tol_primal=tol, max_iter=max_iter, storage=storage,
                                       fused=fused), with_state=False)
    bytes_it = prof["sweep_bytes"]
    line(cfg, m=m, n=n, reg=reg.name(), storage=storage, fused=fused,
         iters_per_s=1e3 / ms_it, ms_per_iter=ms_it, sweep_ms=prof["sweep_ms"],
         reduce_ms=prof["reduce_ms"], update_ms=prof["update_ms"],
         sweep_GBps=bytes_it / prof["sweep_ms"] / 1e6,
         sweep_frac_of_peak=bytes_it / prof["sweep_ms"] / 1e6 / PEAK,
         iter_frac_of_peak=bytes_it / ms_it / 1e6 / PEAK,
         solve_iterations=rep.iterations, solve_termination=rep.termination.name,
         solve_device_s=rep.device_ms / 1e3, objective=rep.objective)
    eng.close()


def run_gl(cfg, m, n, classes, lam, storage, iters, tol=1e-4, max_iter=20000):
    src, tgt, ls, lt = datagen.adaptation_points(m, n, classes, 0)
    eng = otdr.Engine(m, n, storage)
    eng.build_sqdist_cost(src, tgt, datagen.uniform(m), datagen.uniform(n))
    eng.set_regularizer(otdr.GroupLassoReg(lam, otdr.column_class_blocks(ls, n)))
    eng.set_state()
    rho = otdr.default_stepsize(m, n)
    ms_it, prof = steady(eng, rho, iters)
    eng.set_state()
    rep = eng.solve(otdr.SolverOptions(tol_primal=tol, max_iter=max_iter, storage=storage),
                    with_state=False)
    alg = 12.0 * m * n if storage == "f32" else 24.0 * m * n
    line(cfg, m=m, n=n, classes=classes, reg=f"gl:lambda={lam:g}", storage=storage,
         iters_per_s=1e3 / ms_it, ms_per_iter=ms_it, sweep_ms=prof["sweep_ms"],
         sweep_GBps_algorithmic=alg / prof["sweep_ms"] / 1e6,
         sweep_frac_of_peak=alg / prof["sweep_ms"] / 1e6 / PEAK,
         solve_iterations=rep.iterations, solve_termination=rep.termination.name,
         solve_device_s=rep.device_ms / 1e3, objective=rep.objective)
    eng.close()


def run_batched(cfg, B, m, storage, tol=1e-4):
    """One launch: each problem resident in a thread-block cluster."""
    alpha = 5e-3 * (2 * m)
    src = np.empty((B, m, 2))
    tgt = np.empty((B, m, 2))
    for b in range(B):
        src[b], tgt[b] = datagen.gaussian_points(m, m, b)
    ps = np.full((B, m), 1.0 / m)
    be = otdr.BatchEngine(B, m, m, storage)
    be.build_sqdist_costs(src, tgt, ps, ps)
    be.set_regularizer(otdr.QuadraticReg(alpha))
    opt = otdr.SolverOptions(tol_primal=tol, max_iter=20000, storage=storage)
    be.solve(opt)  # warm-up
    t0 = time.perf_counter()
    reps = be.solve(opt)
    wall = time.perf_counter() - t0
    total = sum(r.iterations for r in reps)
    line(cfg, B=B, m=m, n=m, storage=storage, mode=("batched cluster-resident (one launch)"
                                                     if os.environ.get("OTDR_BATCH") == "resident"
                                                     else "batched CTA-per-problem streaming (one launch)"),
         total_iterations=total, wall_s=wall, device_s=reps[0].device_ms / 1e3,
         problem_iters_per_s=total / (reps[0].device_ms / 1e3), mean_iters=total / B,
         max_iters=max(r.iterations for r in reps),
         all_converged=all(r.termination.name == "Converged" for r in reps))
    be.close()


def run_batched_sequential(cfg, B, m, storage, tol=1e-4):
    alpha = 5e-3 * (2 * m)
    engs = []
    for b in range(B):
        eng = gaussian_engine(m, m, b, storage)
        eng.set_regularizer(otdr.QuadraticReg(alpha))
        engs.append(eng)
    for eng in engs[:2]:
        eng.set_state()
        eng.solve(otdr.SolverOptions(tol_primal=tol, max_iter=20000, storage=storage), with_state=False)
    t0 = time.perf_counter()
    total_it = 0
    dev_ms = 0.0
    for eng in engs:
        eng.set_state()
        r = eng.solve(otdr.SolverOptions(tol_primal=tol, max_iter=20000, storage=storage),
                      with_state=False)
        total_it += r.iterations
        dev_ms += r.device_ms
    wall = time.perf_counter() - t0
    line(cfg, B=B, m=m, n=m, storage=storage, mode="sequential engine solves",
         total_iterations=total_it, wall_s=wall, device_s=dev_ms / 1e3,
         problem_iters_per_s=total_it / wall, mean_iters=total_it / B)
    for eng in engs:
        eng.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--fused", action="store_true")
    a = ap.parse_args()
    for c in a.configs:
        if c == "cfg1":
            for st in ("f32", "f64"):
                run_plain("cfg1", 1000, 1000, otdr.QuadraticReg(10.0), st, 1000, fused=a.fused)
        elif c == "cfg2":
            run_plain("cfg2", 10000, 10000, otdr.ZeroReg(), "f32", a.iters, fused=a.fused)
        elif c == "cfg3":
            for lam in (1e-3, 0.06):
                run_gl("cfg3", 10000, 10000, 10, lam, "f32", a.iters)
        elif c == "cfg4":
            run_plain("cfg4", 40000, 40000, otdr.QuadraticReg(400.0), "f32", max(20, a.iters // 5),
                      fused=a.fused, max_iter=3000)
        elif c == "cfg5":
            run_batched("cfg5", 256, 512, "f32")
        elif c == "cfg5-resident":
            os.environ["OTDR_BATCH"] = "resident"
            run_batched("cfg5", 256, 512, "f32")
            os.environ.pop("OTDR_BATCH")
        elif c == "cfg5-seq":
            run_batched_sequential("cfg5", 256, 512, "f32")
        elif c == "headline":
            run_plain("headline", 20000, 20000, otdr.QuadraticReg(200.0), "f32", a.iters)
        elif c == "headline-fused":
            run_plain("headline", 20000, 20000, otdr.QuadraticReg(200.0), "f32", a.iters, fused=True)


if __name__ == "__main__":
    main()
