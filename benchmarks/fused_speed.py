"""Device time of 200-iteration solves, unfused vs SolverOptions.fused (even/odd),
at the headline shape; fp64 and fp32 storage."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: F401
import paper_2305_18483_b200 as otdr
from paper_2305_18483_b200 import datagen
m = n = 20000
src, tgt = datagen.gaussian_points(m, n, 0)
for storage in ("f64", "f32"):
    eng = otdr.Engine(m, n, storage)
    eng.build_sqdist_cost(src, tgt, datagen.uniform(m), datagen.uniform(n))
    eng.set_regularizer(otdr.QuadraticReg(200.0))
    out = {"storage": storage}
    for fused in (False, True, False, True):
        eng.set_state()
        r = eng.solve(otdr.SolverOptions(max_iter=200, tol_primal=1e-300, fused=fused, storage=storage),
                      with_state=False)
        out["fused" if fused else "plain"] = r.device_ms / 200
    bpe = 24 if storage == "f64" else 12
    out["plain_GBps"] = bpe * m * n / (out["plain"] * 1e-3) / 1e9
    out["fused_alg_GBps"] = (bpe - bpe / 6) * m * n / (out["fused"] * 1e-3) / 1e9
    print(json.dumps(out), flush=True)
    eng.close()
