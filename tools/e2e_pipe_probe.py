"""Prototype: all H2D copies up front on one copy stream, kernels per chunk
wait on their chunk's copy event (no staging reuse)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_01566_b200 as h
from paper_2406_01566_b200 import clusters

c = h.Cluster.from_json(json.dumps(clusters.CONFIGS["het42-70b"]("float")))
e = h.Engine(c)
e.mode = "score"
B = 1_000_000
host = torch.from_numpy(h.generate_host(list(e.kmax), c.num_layers, 1, 0, B, 0)).pin_memory()
hv = torch.empty(B, dtype=torch.float64).pin_memory()
hs = torch.empty(B, dtype=torch.int32).pin_memory()
dpl = torch.empty_like(host, device="cuda")
dv = torch.empty(B, dtype=torch.float64, device="cuda")
ds = torch.empty(B, dtype=torch.int32, device="cuda")
cp = torch.cuda.Stream()
ks = torch.cuda.Stream()
for sizes_name, first in (("ramp16k", 1 << 14), ("flat256k", 1 << 18), ("ramp64k", 1 << 16)):
    bounds = []
    lo, sz = 0, first
    while lo < B:
        n = min(sz, B - lo)
        bounds.append((lo, n))
        lo += n
        sz = min(1 << 18, 2 * sz)
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        evs = []
        with torch.cuda.stream(cp):
            for lo, n in bounds:
                dpl[lo:lo + n].copy_(host[lo:lo + n], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cp)
                evs.append(ev)
        for (lo, n), ev in zip(bounds, evs):
            ks.wait_event(ev)
            e.score_device(dpl[lo].data_ptr(), n, dv[lo].data_ptr(), ds[lo].data_ptr(), True, ks.cuda_stream)
            with torch.cuda.stream(ks):
                hv[lo:lo + n].copy_(dv[lo:lo + n], non_blocking=True)
                hs[lo:lo + n].copy_(ds[lo:lo + n], non_blocking=True)
        ks.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
    print(json.dumps({"schedule": sizes_name, "chunks": len(bounds), "ms": dt}))
torch.cuda.synchronize()
t0 = time.perf_counter()
e.score_device(dpl.data_ptr(), B, dv.data_ptr(), ds.data_ptr(), True, ks.cuda_stream)
ks.synchronize()
print(json.dumps({"device_only_ms": (time.perf_counter() - t0) * 1e3}))
t0 = time.perf_counter()
e.score_best_host_ptr(host.data_ptr(), B, hv.data_ptr(), hs.data_ptr(), True)
print(json.dumps({"score_best_host_ms": (time.perf_counter() - t0) * 1e3}))
