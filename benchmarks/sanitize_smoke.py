"""Small solves through every persistent kernel, for compute-sanitizer
(memcheck / racecheck / synccheck): stream (fp32, fp64, fused), gl_stream,
bstream (batched), resident."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2305_18483_b200 as otdr
from paper_2305_18483_b200 import datagen

os.environ["OTDR_RESIDENT"] = "off"
m, n = 300, 520
src, tgt = datagen.gaussian_points(m, n, 1)
p, q = datagen.uniform(m), datagen.uniform(n)
for storage in ("f32", "f64"):
    for reg in (otdr.QuadraticReg(2.0), otdr.GroupLassoReg(1e-3, otdr.column_class_blocks([i % 3 for i in range(m)], n))):
        for fused in (False, True):
            if fused and isinstance(reg, otdr.GroupLassoReg):
                continue
            eng = otdr.Engine(m, n, storage)
            eng.build_sqdist_cost(src, tgt, p, q)
            eng.set_regularizer(reg)
            eng.set_state()
            r = eng.solve(otdr.SolverOptions(tol_primal=1e-5, max_iter=40, fused=fused, storage=storage), with_state=False)
            print(storage, reg.name(), fused, eng.solve_path(), r.iterations, r.objective, flush=True)
            eng.close()
os.environ["OTDR_RESIDENT"] = "on"
B = 4
srcb = np.stack([datagen.gaussian_points(128, 128, b)[0] for b in range(B)])
tgtb = np.stack([datagen.gaussian_points(128, 128, b)[1] for b in range(B)])
be = otdr.BatchEngine(B, 128, 128, "f32")
be.build_sqdist_costs(srcb, tgtb, np.full((B, 128), 1 / 128), np.full((B, 128), 1 / 128))
be.set_regularizer(otdr.QuadraticReg(1.28))
print("batch", [x.iterations for x in be.solve(otdr.SolverOptions(tol_primal=1e-4, max_iter=50))])
be.close()
eng = otdr.Engine(200, 150, "f32")
eng.build_sqdist_cost(src[:200], tgt[:150], datagen.uniform(200), datagen.uniform(150))
eng.set_regularizer(otdr.QuadraticReg(1.0))
eng.set_state()
print("resident", eng.solve_path(), eng.solve(otdr.SolverOptions(max_iter=30, tol_primal=1e-9), with_state=False).iterations)
