"""Phase timestamps of the streaming solve kernel (OTDR_STREAM_TRACE=1).

  OTDR_STREAM_TRACE=1 python benchmarks/stream_trace.py [m [n [peer1]]]
(m x n band of the 20000^2 headline points; peer1 = 1-rank peer group, i.e.
the row-sharded kernel with the in-kernel exchange)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: F401
import paper_2305_18483_b200 as otdr
from paper_2305_18483_b200 import datagen
m = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
n = int(sys.argv[2]) if len(sys.argv) > 2 else m
eng = otdr.Engine(m, n, "f32")
if len(sys.argv) > 3 and sys.argv[3] == "peer1":
    otdr.link_local([eng])
src, tgt = datagen.gaussian_points(max(m, n), n, 0)
eng.build_sqdist_cost(src[:m], tgt, datagen.uniform(m), datagen.uniform(n))
eng.set_regularizer(otdr.QuadraticReg(5e-3 * 2 * max(m, n)))
eng.set_state()
rho = otdr.default_stepsize(max(m, n), n)
for _ in range(3):
    eng.step(rho, 6)
