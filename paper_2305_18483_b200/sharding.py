"""Row sharding of the plan across GPUs (one process per GPU).

Rank r owns a contiguous band of plan rows. Per DR iteration each rank sweeps
its band (row sums complete locally), then ONE ncclAllReduce of the n+3 vector
[column sums | sum r | sum r^2 | sum X] gives every rank the global column sums
and residual scalars; every rank then updates the replicated column-side
vectors (psi, b, s) and its own rows of (phi, a) identically.

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


def open_sharded_engine(dist, m: int, n: int, storage: str = "f32", device: int = 0,
                        labels: Optional[Sequence[int]] = None) -> Tuple[Engine, int, int]:
    """Engine over this rank's band (collective: every rank must call it)."""
    rank, world = dist.get_rank(), dist.get_world_size()
    lo, hi = row_bands(m, world, labels)[rank]
    nid = broadcast_nccl_id(dist, rank)
    return Engine(m, n, storage, device=device, shard=Shard(rank, world, lo, hi, nid)), lo, hi
