"""Phase timestamps of the streaming solve kernel (OTDR_STREAM_TRACE=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: F401
import paper_2305_18483_b200 as otdr
from paper_2305_18483_b200 import datagen
m = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
eng = otdr.Engine(m, m, "f32")
src, tgt = datagen.gaussian_points(m, m, 0)
eng.build_sqdist_cost(src, tgt, datagen.uniform(m), datagen.uniform(m))
eng.set_regularizer(otdr.QuadraticReg(5e-3 * 2 * m))
eng.set_state()
rho = otdr.default_stepsize(m, m)
for _ in range(3):
    eng.step(rho, 6)
