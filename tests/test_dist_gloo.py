"""CPU, world_size 2 (gloo): the multi-rank sharding + argmax reduction that
bench.py runs over NCCL on GPUs."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2406_01566_b200.dist import gather_best, owner_of, pack_record, reduce_best, shard_range, strong_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, values, q, strong=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    if strong:  # bench.py's default: the global batch split over the ranks
        lo, hi = strong_range(len(values), world, rank)
    else:
        lo, hi = shard_range(len(values) // world, rank)
    local = values[lo:hi]
    ok = local > 0
    if ok.any():
        i = int(np.argmax(np.where(ok, local, -1.0)))
        rec = pack_record(float(local[i]), lo + i)
    else:
        rec = pack_record(0.0, -1)
    q.put((rank, gather_best(rec, world)))
    dist.destroy_process_group()


def _run(values, world=2, strong=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, values, q, strong)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return dict(res)


def _first_max(values):
    ok = values > 0
    if not ok.any():
        return 0.0, -1
    i = int(np.argmax(np.where(ok, values, -1.0)))
    return float(values[i]), i


@pytest.mark.parametrize("case", ["random", "tie_across_ranks", "all_zero"])
def test_two_rank_argmax_equals_global_first_max(case):
    rng = np.random.default_rng(5)
    v = rng.random(64) * 100
    if case == "tie_across_ranks":
        v[:] = 1.0
        v[40] = 7.0
        v[10] = 7.0  # rank 0 and rank 1 tie: min global index (10) must win
    if case == "all_zero":
        v[:] = 0.0
    res = _run(v)
    want = _first_max(v)
    assert res[0] == want and res[1] == want


@pytest.mark.parametrize("world", [2, 3])
def test_strong_scaling_shards_reduce_to_the_global_first_max(world):
    rng = np.random.default_rng(11)
    v = np.round(rng.random(61) * 10)  # ties across uneven shards
    res = _run(v, world=world, strong=True)
    want = _first_max(v)
    assert all(res[r] == want for r in range(world))


def test_reduce_best_rules():
    assert reduce_best([(3.0, 5), (3.0, 2), (1.0, 0)]) == (3.0, 2)
    assert reduce_best([(0.0, -1), (0.0, -1)]) == (0.0, -1)
    assert shard_range(1000, 3) == (3000, 4000)
    assert [strong_range(10, 4, r) for r in range(4)] == [(0, 2), (2, 5), (5, 7), (7, 10)]
    starts = [strong_range(10, 4, r)[0] for r in range(4)]
    assert [owner_of(i, starts) for i in (0, 1, 2, 4, 5, 9)] == [0, 0, 1, 1, 2, 3]
    assert owner_of(-1, starts) == -1
    assert pack_record(2.5, 7).tolist()[1] == 7


def _share_worker(rank, world, port, q):
    from paper_2406_01566_b200.dist import share_winner

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    index = 137  # owned by rank 1 (weak shards of 100)
    owner = owner_of(index, [0, 100])
    row = flows = None
    if rank == owner:
        row = np.arange(2 * 7, dtype=np.int16).reshape(7, 2)
        flows = np.linspace(0.5, 3.5, 11)
    r, f = share_winner(owner, row, flows, 7)
    assert share_winner(-1) is None  # no valid candidate anywhere: nothing to broadcast
    q.put((rank, (r.tolist(), f.tolist())))
    dist.destroy_process_group()


def _group_worker(rank, world, port, q):
    from paper_2406_01566_b200.dist import share_winner

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = dist.new_group([1, 2])  # group rank 0 = global rank 1
    out = None
    if rank in (1, 2):
        row = np.full((3, 2), 5, np.int16) if rank == 1 else None
        flows = np.array([1.25, 2.5]) if rank == 1 else None
        r, f = share_winner(0, row, flows, 3, group=g)
        out = (r.tolist(), f.tolist())
    q.put((rank, out))
    dist.destroy_process_group()


def test_winner_broadcast_maps_group_ranks_to_global_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_group_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = ([[5, 5]] * 3, [1.25, 2.5])
    assert res[0] is None and res[1] == want and res[2] == want


def test_winner_plan_is_broadcast_from_its_owner():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_share_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = (np.arange(14).reshape(7, 2).tolist(), np.linspace(0.5, 3.5, 11).tolist())
    assert res[0] == want and res[1] == want
