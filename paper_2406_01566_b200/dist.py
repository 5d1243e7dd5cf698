"""Multi-rank plumbing for candidate sharding (one process per GPU).

The path partitions: rank r owns global candidate indices [r*B, (r+1)*B)
(weak scaling) and needs no input exchange.  The only collective is the
argmax: each rank's 16-byte record (value bits, global index) is all-gathered
and reduced deterministically — max value, then min index — which reproduces
the strict first-wins `v > best` of tests/oracles/enumerate.hpp:59 over the
global enumeration order.
"""

from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np


def shard_range(per_rank: int, rank: int) -> Tuple[int, int]:
    """Global index range of `rank` under weak scaling."""
    return rank * per_rank, (rank + 1) * per_rank


def reduce_best(records: Sequence[Tuple[float, int]]) -> Tuple[float, int]:
    """(value, index) records -> the first maximum; (0.0, -1) if none is valid."""
    best_v, best_i = 0.0, -1
    for v, i in records:
        if i < 0:
            continue
        if best_i < 0 or v > best_v or (v == best_v and i < best_i):
            best_v, best_i = v, i
    return best_v, best_i


def pack_record(value: float, index: int):
    """16-byte int64 pair: float64 bits + global index."""
    import torch
    rec = torch.empty(2, dtype=torch.int64)
    rec[0] = int(np.array([value], np.float64).view(np.int64)[0])
    rec[1] = index
    return rec


def unpack_records(gathered) -> List[Tuple[float, int]]:
    g = gathered.reshape(-1, 2).cpu().numpy()
    return [(float(g[r, 0:1].view(np.float64)[0]), int(g[r, 1])) for r in range(g.shape[0])]


def gather_best(rec, world: int, group=None) -> Tuple[float, int]:
    """All-gather each rank's packed record (a 2-element int64 tensor on the
    backend's device) and reduce it identically on every rank."""
    import torch
    import torch.distributed as dist
    out = torch.empty(2 * world, dtype=torch.int64, device=rec.device)
    dist.all_gather_into_tensor(out, rec, group=group)
    return reduce_best(unpack_records(out))
