"""Multi-rank plumbing for candidate sharding (one process per GPU).

The path partitions: every candidate is independent, so a rank scores a
contiguous range of global candidate indices and needs no input exchange.
Strong scaling splits a global batch G as [r*G/N, (r+1)*G/N); weak scaling
gives every rank its own `per_rank` candidates [r*B, (r+1)*B).  The only
collective is the argmax: each rank's 16-byte record (value bits, global index)
is all-gathered and reduced deterministically — max value, then min index —
which reproduces the strict first-wins `v > best` of
tests/oracles/enumerate.hpp:59 over the global enumeration order.
"""

from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np


def shard_range(per_rank: int, rank: int) -> Tuple[int, int]:
    """Global index range of `rank` under weak scaling."""
    return rank * per_rank, (rank + 1) * per_rank


def strong_range(total: int, world: int, rank: int) -> Tuple[int, int]:
    """Global index range of `rank` when `total` candidates are split over
    `world` ranks (strong scaling; sizes differ by at most one)."""
    return rank * total // world, (rank + 1) * total // world


def owner_of(index: int, starts: Sequence[int]) -> int:
    """The rank whose range holds global `index`, given every rank's first
    index (ascending); -1 for a negative index (no valid candidate)."""
    if index < 0:
        return -1
    owner = 0
    for r, s in enumerate(starts):
        if s <= index:
            owner = r
    return owner


def reduce_best(records: Sequence[Tuple[float, int]]) -> Tuple[float, int]:
    """(value, index) records -> the first maximum; (0.0, -1) if none is valid."""
    best_v, best_i = 0.0, -1
    for v, i in records:
        if i < 0:
            continue
        if best_i < 0 or v > best_v or (v == best_v and i < best_i):
            best_v, best_i = v, i
    return best_v, best_i


def pack_record(value: float, index: int, device=None):
    """16-byte int64 pair: float64 bits + global index, on `device` (the
    backend's device: CUDA for NCCL, CPU for gloo)."""
    import torch
    rec = torch.tensor([int(np.array([value], np.float64).view(np.int64)[0]), int(index)], dtype=torch.int64)
    return rec if device is None else rec.to(device)


def unpack_records(gathered) -> List[Tuple[float, int]]:
    g = gathered.reshape(-1, 2).cpu().numpy()
    return [(float(g[r, 0:1].view(np.float64)[0]), int(g[r, 1])) for r in range(g.shape[0])]


def gather_best(rec, world: int, group=None) -> Tuple[float, int]:
    """All-gather each rank's packed record (a 2-element int64 tensor on the
    backend's device, see pack_record) and reduce it identically on every rank."""
    import torch
    import torch.distributed as dist
    out = torch.empty(2 * world, dtype=torch.int64, device=rec.device)
    dist.all_gather_into_tensor(out, rec, group=group)
    return reduce_best(unpack_records(out))


def share_winner(owner: int, row=None, flows=None, n_nodes: Optional[int] = None, group=None):
    """after the argmax, rank `owner` (a rank within
    `group`; see owner_of) broadcasts the winning placement row (int16 [N][2])
    and its PARITY per-edge flows (float64 [E], reference edge order) so that
    every rank can materialise the plan and route without re-scoring.  `row`
    and `flows` are read on the owner only.  -> (row int16 [N][2], flows
    float64 [E]) on every rank, as CPU numpy arrays; None when owner < 0 (no
    valid candidate anywhere)."""
    import torch
    import torch.distributed as dist
    if owner < 0:
        return None
    me = dist.get_rank(group)
    src = owner if group is None else dist.get_global_rank(group, owner)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else torch.device("cpu")
    meta = torch.zeros(2, dtype=torch.int64, device=dev)
    if me == owner:
        meta[0] = int(np.asarray(row).size)
        meta[1] = int(np.asarray(flows).size)
    dist.broadcast(meta, src=src, group=group)
    nr, ne = int(meta[0]), int(meta[1])
    r = torch.zeros(nr, dtype=torch.int32, device=dev)  # gloo has no int16 collectives
    f = torch.zeros(ne, dtype=torch.float64, device=dev)
    if me == owner:
        r.copy_(torch.from_numpy(np.ascontiguousarray(row, np.int32).reshape(-1)))
        f.copy_(torch.from_numpy(np.ascontiguousarray(flows, np.float64).reshape(-1)))
    dist.broadcast(r, src=src, group=group)
    dist.broadcast(f, src=src, group=group)
    out_row = r.cpu().numpy().astype(np.int16).reshape(-1, 2)
    if n_nodes is not None and out_row.shape[0] != n_nodes:
        raise ValueError(f"broadcast row has {out_row.shape[0]} nodes, expected {n_nodes}")
    return out_row, f.cpu().numpy()
