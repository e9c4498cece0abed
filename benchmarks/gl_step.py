"""cfg3 (10000^2, 10 classes, lambda 1e-3, fp32): warm up, then ONE
gl_stream_kernel launch of 2 DR iterations (for ncu -k regex:gl_stream -s 1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: F401
import paper_2305_18483_b200 as otdr
from paper_2305_18483_b200 import datagen
m = n = 10000
src, tgt, ls, lt = datagen.adaptation_points(m, n, 10, 0)
eng = otdr.Engine(m, n, "f32")
eng.build_sqdist_cost(src, tgt, datagen.uniform(m), datagen.uniform(n))
eng.set_regularizer(otdr.GroupLassoReg(1e-3, otdr.column_class_blocks(ls, n)))
eng.set_state()
rho = otdr.default_stepsize(m, n)
eng.step(rho, 3)
eng.step(rho, 2)
print(eng.solve_path())
