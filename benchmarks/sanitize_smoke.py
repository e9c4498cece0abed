"""Small solves through every device loop, for compute-sanitizer
(memcheck / racecheck / synccheck):

  * streaming solve kernels: tstream_kernel (TMA producer warp, fp32),
    stream_kernel (per-thread cp.async: fp64, fp32 with
    OTDR_STREAM_KERNEL=async, fused even/odd)
  * gl_stream_kernel (group lasso), the CUDA-graph loop (sweep / reduce /
    update + certificate, trace), the on-chip resident kernel
  * the batched kernels (bstream, cluster-resident)
  * the row-sharded peer exchange inside the streaming kernel: 2 rank contexts
    of this process linked over peer memory (--peer; the two ranks' kernels
    spin on each other's flags, so this part needs concurrent kernels and
    hangs under the sanitizers' serialized launches -- run it without them)

  compute-sanitizer --tool memcheck python benchmarks/sanitize_smoke.py
"""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2305_18483_b200 as otdr  # noqa: E402
from paper_2305_18483_b200 import datagen  # noqa: E402

m, n = 300, 520
src, tgt = datagen.gaussian_points(m, n, 1)
p, q = datagen.uniform(m), datagen.uniform(n)


# --no-conditional: racecheck aborts on CUDA graphs with conditional (WHILE)
# nodes, which solve() uses on the graph loop (traces, OTDR_STREAM=off); with
# this flag those cases run step() (plain chunk graphs) instead.
NO_COND = "--no-conditional" in sys.argv


def run(storage, reg, env=None, fused=False, trace=False):
    env = env or {}
    graph_loop = trace or env.get("OTDR_STREAM") == "off"
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        eng = otdr.Engine(m, n, storage)
        eng.build_sqdist_cost(src, tgt, p, q)
        eng.set_regularizer(reg)
        eng.set_state()
        if NO_COND and graph_loop:
            os.environ["OTDR_STREAM"] = "off"
            eng.close()
            eng = otdr.Engine(m, n, storage)
            eng.build_sqdist_cost(src, tgt, p, q)
            eng.set_regularizer(reg)
            eng.set_state()
            eng.step(otdr.default_stepsize(m, n), 40)
            print(storage, reg.name(), env, "graph loop via step()", eng.kernel_name(),
                  eng.get_state(with_plan=False).k, flush=True)
            os.environ.pop("OTDR_STREAM")
            if "OTDR_STREAM" in env:
                os.environ["OTDR_STREAM"] = env["OTDR_STREAM"]
            eng.close()
            return
        r = eng.solve(otdr.SolverOptions(tol_primal=1e-5, max_iter=40, fused=fused, storage=storage,
                                         record_trace=trace, check_every=10 if trace else 1),
                      with_state=False)
        print(storage, reg.name(), env, "fused" if fused else "", "trace" if trace else "",
              eng.kernel_name(), r.iterations, r.objective, flush=True)
        eng.close()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


os.environ["OTDR_RESIDENT"] = "off"
quad = otdr.QuadraticReg(2.0)
gl = otdr.GroupLassoReg(1e-3, otdr.column_class_blocks([i % 3 for i in range(m)], n))
for storage in ("f32", "f64"):
    run(storage, quad)
    run(storage, otdr.ZeroReg())
    run(storage, quad, fused=True)
    run(storage, gl)
    run(storage, quad, trace=True)  # graph loop with certificate kernels
run("f32", quad, {"OTDR_STREAM_KERNEL": "async"})
run("f32", quad, {"OTDR_STREAM": "off"})

# row-sharded: 2 rank contexts on this GPU, in-kernel peer exchange
if "--peer" in sys.argv:
    os.environ["OTDR_STREAM_GRID"] = "64"
    C = datagen.squared_distance_cost(src, tgt)
    C /= C.max()
    engs = []
    for rank, (lo, hi) in enumerate(((0, 150), (150, 300))):
        e = otdr.Engine(m, n, "f32", shard=otdr.Shard(rank, 2, lo, hi, None))
        e.set_problem(C[lo:hi], p[lo:hi], q)  # setup (allocations) before linking, like the tests
        e.set_regularizer(quad)
        engs.append(e)
    otdr.link_local(engs)

    def rank_run(e):  # make_state sums and the steps are collective: one thread per rank
        e.set_state()
        e.step(otdr.default_stepsize(m, n), 20)

    ths = [threading.Thread(target=rank_run, args=(e,)) for e in engs]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    print("peer exchange", [e.get_state(with_plan=False).k for e in engs], flush=True)
    for e in engs:
        e.close()
    os.environ.pop("OTDR_STREAM_GRID")

os.environ["OTDR_RESIDENT"] = "on"
B = 4
srcb = np.stack([datagen.gaussian_points(128, 128, b)[0] for b in range(B)])
tgtb = np.stack([datagen.gaussian_points(128, 128, b)[1] for b in range(B)])
for mode in ("stream", "resident"):
    os.environ["OTDR_BATCH"] = mode
    be = otdr.BatchEngine(B, 128, 128, "f32")
    be.build_sqdist_costs(srcb, tgtb, np.full((B, 128), 1 / 128), np.full((B, 128), 1 / 128))
    be.set_regularizer(otdr.QuadraticReg(1.28))
    print("batch", mode, [x.iterations for x in be.solve(otdr.SolverOptions(tol_primal=1e-4, max_iter=50))])
    be.close()
eng = otdr.Engine(200, 150, "f32")
eng.build_sqdist_cost(src[:200], tgt[:150], datagen.uniform(200), datagen.uniform(150))
eng.set_regularizer(otdr.QuadraticReg(1.0))
eng.set_state()
print("resident", eng.kernel_name(), eng.solve(otdr.SolverOptions(max_iter=30, tol_primal=1e-9), with_state=False).iterations)
