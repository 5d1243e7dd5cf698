"""Library-level multi-GPU (csrc/multi.cu).

* MultiEngine: one process, several device contexts; a host batch is split
  into contiguous shards and the first maxima merged in index order — equal to
  one engine scoring the whole batch (runs on one GPU too, with two contexts on
  device 0).
* helio_gpu_argmax_ranked: one process per GPU, the 16-byte (value, index)
  records all-gathered over an NCCL communicator the library creates
  (nccl_unique_id / NcclComm) — equal to the global first maximum.  Needs two
  GPUs (gpurun --gpus 2).  The same reduction rule is covered on CPU by the
  gloo tests in tests/test_dist_gloo.py.
"""

import json
import os
import socket

import numpy as np
import pytest

import paper_2406_01566_b200 as h
from paper_2406_01566_b200 import clusters
from _support import bits

pytestmark = pytest.mark.gpu


def _gpus():
    import torch
    return torch.cuda.device_count()


def _first_max(v, st):
    ok = (st == 0) & (v > 0)
    if not ok.any():
        return 0.0, -1
    i = int(np.argmax(np.where(ok, v, -1.0)))
    return float(v[i]), i


@pytest.mark.parametrize("mode", ["parity", "score"])
def test_multi_engine_equals_one_engine(mode):
    d = clusters.CONFIGS["het42-70b"]("float")
    c = h.Cluster.from_json(json.dumps(d))
    e = h.Engine(c)
    e.mode = mode
    devs = [0, 1] if _gpus() >= 2 else [0, 0]
    m = h.MultiEngine(c, devs)
    m.mode = mode
    assert m.count == 2 and list(m.kmax) == list(e.kmax)
    rows = h.generate_host(list(e.kmax), c.num_layers, 99, 0, 50_001, 20_000)
    rows[::997, 3] = (0, 80)  # invalid rows (exceed k_i) keep their status
    v1, s1 = e.score(rows)
    v2, s2, best, idx = m.score_best(rows)
    assert np.array_equal(bits(v1), bits(v2)) and np.array_equal(s1, s2)
    assert (best, idx) == _first_max(v1, s1)
    # ties across the shard boundary: the lower global index wins
    tie = np.repeat(rows[1:2], 6, axis=0)
    assert s1[1] == 0 and v1[1] > 0
    _, _, bt, it = m.score_best(tie)
    assert it == 0 and bt == v1[1]


def test_multi_device_sampled_search_equals_one_device():
    """helio_gpu_multi_sampled_search splits every round's mutants over the
    devices and merges first maxima in index order: same rounds, same moves,
    same placement and value bits as Engine.sampled_search on one device."""
    d = clusters.CONFIGS["het42-70b"]("float")
    c = h.Cluster.from_json(json.dumps(d))
    e = h.Engine(c)
    e.mode = "score"
    devs = [0, 1] if _gpus() >= 2 else [0, 0]
    m = h.MultiEngine(c, devs)
    m.mode = "score"
    placement, _ = h.heuristic_placement(c, "petals")
    seed = h.placement_rows(c, [{k: tuple(v) for k, v in placement.items()}])[0]
    v1, r1, i1, s1 = e.sampled_search(seed, True, 6, 1 << 16, 2, 7)
    v2, r2, i2, s2 = m.sampled_search(seed, True, 6, 1 << 16, 2, 7)
    assert bits([v1])[0] == bits([v2])[0] and np.array_equal(r1, r2) and (i1, s1) == (i2, s2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ranked_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)  # only to ship the NCCL id
    uid = [h.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = h.NcclComm(uid[0], world, rank, rank)
    d = clusters.CONFIGS["het42-70b"]("float")
    c = h.Cluster.from_json(json.dumps(d))
    e = h.Engine(c, device=rank)
    e.mode = "score"
    G = 200_000
    lo, hi = rank * G // world, (rank + 1) * G // world
    dev = torch.device("cuda", rank)
    s = torch.cuda.Stream(dev)
    pl = torch.empty((hi - lo, e.num_nodes, 2), dtype=torch.int16, device=dev)
    e.generate_device(7, lo, hi - lo, 0, pl.data_ptr(), s.cuda_stream)
    v = torch.empty(hi - lo, dtype=torch.float64, device=dev)
    st = torch.empty(hi - lo, dtype=torch.int32, device=dev)
    best = torch.empty(1, dtype=torch.float64, device=dev)
    idx = torch.empty(1, dtype=torch.int64, device=dev)
    e.score_device(pl.data_ptr(), hi - lo, v.data_ptr(), st.data_ptr(), True, s.cuda_stream)
    e.argmax_ranked(v.data_ptr(), st.data_ptr(), hi - lo, lo, best.data_ptr(), idx.data_ptr(), comm.handle,
                    s.cuda_stream)
    s.synchronize()
    q.put((rank, float(best.item()), int(idx.item()), v.cpu().numpy(), st.cpu().numpy()))
    dist.barrier()
    del comm
    dist.destroy_process_group()


@pytest.mark.skipif(_gpus() < 2, reason="needs two GPUs (gpurun --gpus 2)")
def test_ranked_argmax_over_nccl_equals_global_first_max():
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ranked_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in procs), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    v = np.concatenate([r[3] for r in res])
    st = np.concatenate([r[4] for r in res])
    want = _first_max(v, st)
    for r in res:
        assert (r[1], r[2]) == want
