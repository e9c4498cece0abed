"""Row sharding of the plan across GPUs (one process per GPU).

Rank r owns a contiguous band of plan rows. Per DR iteration each rank sweeps
its band (row sums complete locally) and the n+3 vector [column sums | sum r |
sum r^2 | sum X] is all-reduced; every rank then updates the replicated
column-side vectors (psi, b, s) and its own rows of (phi, a) identically
(SURVEY §8(e)). With peers linked (connect_peers, CUDA IPC) the exchange runs
inside the streaming kernel over NVLink: each stripe's column sums are stored
into every rank's receive buffer as soon as the stripe is swept (overlapped
with the rest of the sweep), and epoch flags at system scope order the fold.
Without a peer link, one ncclAllReduce per iteration between kernels.

Group lasso: a group is (column, class), so a class's rows must all live on
one rank for its norms to stay local -- bands are cut at class boundaries and a
class split across bands is rejected (Unsupported), never silently mis-solved.
"""
from __future__ import annotations

import ctypes as ct
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native as nat
from .otdr import Engine, Shard, Unsupported


def row_bands(m: int, world: int, labels: Optional[Sequence[int]] = None) -> List[Tuple[int, int]]:
    """Contiguous row bands, balanced; cut only at class boundaries when
    `labels` (group-lasso row classes, -1 = ungrouped) are given."""
    if world < 1:
        raise ValueError("world must be >= 1")
    even = [(m * r // world, m * (r + 1) // world) for r in range(world)]
    if labels is None:
        return even
    lab = np.asarray(labels).reshape(-1)
    if lab.shape[0] != m:
        raise ValueError("labels must have one entry per row")
    # allowed cut points: row indices where the class changes, plus 0 and m;
    # every grouped class must be one contiguous run.
    cuts = [0] + [i for i in range(1, m) if lab[i] != lab[i - 1]] + [m]
    seen = set()
    for a, b in zip(cuts[:-1], cuts[1:]):
        c = int(lab[a])
        if c >= 0:
            if c in seen:
                raise Unsupported(f"class {c} is not contiguous: its groups would span ranks")
            seen.add(c)
    # ungrouped rows (-1) may be cut anywhere
    allowed = set(cuts)
    allowed.update(i for i in range(m) if lab[i] < 0 or (i > 0 and lab[i - 1] < 0))
    allowed = sorted(allowed)
    bounds = [0]
    for r in range(1, world):
        target = m * r // world
        best = min((x for x in allowed if x >= bounds[-1]), key=lambda x: (abs(x - target), x))
        bounds.append(best)
    bounds.append(m)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def nccl_unique_id() -> bytes:
    raw = ct.create_string_buffer(128)
    rc = nat.lib().otdr_dev_nccl_unique_id(raw)
    if rc:
        raise RuntimeError("ncclGetUniqueId failed (libnccl.so.2 not loadable?)")
    return raw.raw


def broadcast_nccl_id(dist, rank: int) -> bytes:
    """Rank 0 creates the NCCL id; torch.distributed (any backend) broadcasts it."""
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def connect_peers(dist, eng: Engine, device: Optional[int] = None) -> bool:
    """All-gather every rank's receive-buffer IPC handle and import them, so
    the solve loop exchanges column sums over NVLink peer memory inside the
    streaming kernel (collective). Returns False -- the context keeps its NCCL
    exchange -- when some pair of the ranks' GPUs has no peer access; raises
    if a handle that should map does not."""
    world = dist.get_world_size()
    ok = 1
    try:
        import torch

        dev = torch.cuda.current_device() if device is None else device
        devs = [None] * world
        dist.all_gather_object(devs, dev)
        ok = int(all(d == dev or torch.cuda.can_device_access_peer(dev, d) for d in devs))
    except Exception:  # no torch / no CUDA runtime view: let the import decide
        ok = 1
    flags = [None] * world
    dist.all_gather_object(flags, ok)
    if not all(flags):
        return False
    handles = [None] * world
    dist.all_gather_object(handles, eng.peer_export())
    err = ""
    try:
        eng.peer_import(handles)
    except Exception as e:  # pragma: no cover - hardware dependent
        err = str(e) or type(e).__name__
    errs = [None] * world
    dist.all_gather_object(errs, err)
    if any(errs):
        raise RuntimeError("peer-memory exchange could not be set up: " + "; ".join(e for e in errs if e))
    return True


def open_sharded_engine(dist, m: int, n: int, storage: str = "f32", device: int = 0,
                        labels: Optional[Sequence[int]] = None,
                        peers: bool = True) -> Tuple[Engine, int, int]:
    """Engine over this rank's band (collective: every rank must call it).
    peers=True links the ranks' receive buffers for the in-kernel exchange."""
    rank, world = dist.get_rank(), dist.get_world_size()
    lo, hi = row_bands(m, world, labels)[rank]
    nid = broadcast_nccl_id(dist, rank)
    eng = Engine(m, n, storage, device=device, shard=Shard(rank, world, lo, hi, nid))
    if peers and world > 1:
        connect_peers(dist, eng)
    return eng, lo, hi
