import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import numpy as np
import paper_2305_18483_b200 as otdr
import pyoracle as ora
m, n = int(sys.argv[1]), int(sys.argv[2])
C, p, q, *_ = ora.gaussian_problem(m, n, 5 + m)
labels = [i % 3 for i in range(m)]
eng = otdr.Engine(m, n, sys.argv[3])
eng.set_problem(C, p, q)
eng.set_regularizer(otdr.GroupLassoReg(0.02, otdr.column_class_blocks(labels, n)))
eng.set_state()
eng.step(ora.default_stepsize(m, n), 3)
print("ok", eng.get_state().X.sum())
