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


def share_winner(index: int, per_rank: int, row=None, flows=None, group=None):
    """after the argmax, the rank that owns global
    candidate `index` broadcasts the winning placement row (int16 [N][2]) and
    its PARITY per-edge flows (float64 [E], reference edge order) so that every
    rank can materialise the plan and route without re-scoring.  `row` and
    `flows` are read on the owner only.  -> (row int16 [N][2], flows float64 [E])
    on every rank, as CPU numpy arrays."""
    import torch
    import torch.distributed as dist
    owner = index // per_rank
    me = dist.get_rank(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else torch.device("cpu")
    meta = torch.zeros(2, dtype=torch.int64, device=dev)
    if me == owner:
        meta[0] = int(np.asarray(row).size)
        meta[1] = int(np.asarray(flows).size)
    dist.broadcast(meta, src=owner, group=group)
    nr, ne = int(meta[0]), int(meta[1])
    r = torch.zeros(nr, dtype=torch.int32, device=dev)  # gloo has no int16 collectives
    f = torch.zeros(ne, dtype=torch.float64, device=dev)
    if me == owner:
        r.copy_(torch.from_numpy(np.ascontiguousarray(row, np.int32).reshape(-1)))
        f.copy_(torch.from_numpy(np.ascontiguousarray(flows, np.float64).reshape(-1)))
    dist.broadcast(r, src=owner, group=group)
    dist.broadcast(f, src=owner, group=group)
    return r.cpu().numpy().astype(np.int16).reshape(-1, 2), f.cpu().numpy()
