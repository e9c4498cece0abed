"""Two processes on one GPU as the two ranks of a row-sharded run, exchanging
over CUDA IPC peer memory inside the streaming kernel (the multi-GPU path of
bench.py --gpus N, minus NVLink). The two contexts time-slice the GPU."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.timeout(300, method="thread")
def test_peer_ipc_two_processes():
    env = dict(os.environ, OTDR_STREAM_GRID="64")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "_peer_ipc_worker.py")]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=240)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    assert "PEER_IPC_OK" in out.stdout, out.stdout[-2000:]


@pytest.mark.timeout(400, method="thread")
def test_bench_two_ranks_rehearsal():
    """bench.py's torchrun N = 2 path (row sharding, in-kernel exchange,
    time to tolerance, max-over-ranks timing, one JSON line from rank 0) with
    both ranks on cuda:0 (OTDR_BENCH_SHARED_GPU=1: gloo, no NCCL id)."""
    import json

    env = dict(os.environ, OTDR_STREAM_GRID="64", OTDR_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-e2e"]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=360, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = lines[0]
    assert d["n_gpus"] == 2 and d["steps"] == 3 and d["value"] > 0 and "rehearsal" in d
    assert d["config"]["parallelism"] == "row-shard x2"
    assert d["time_to_tol"]["termination"] == "Converged"
    assert abs(d["time_to_tol"]["iterations"] - 1154) <= 1  # the one-GPU bench: 1154
