"""Where the e2e time goes: device-only scoring vs host-buffer scoring vs a bare H2D."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_01566_b200 as h
from paper_2406_01566_b200 import clusters

c = h.Cluster.from_json(json.dumps(clusters.CONFIGS["het42-70b"]("float")))
e = h.Engine(c)
e.mode = "score"
B = 1_000_000
N = e.num_nodes
host = torch.from_numpy(h.generate_host(list(e.kmax), c.num_layers, 1, 0, B, 0)).pin_memory()
hv = torch.empty(B, dtype=torch.float64).pin_memory()
hs = torch.empty(B, dtype=torch.int32).pin_memory()
dpl = host.cuda()
dv = torch.empty(B, dtype=torch.float64, device="cuda")
ds = torch.empty(B, dtype=torch.int32, device="cuda")
s = torch.cuda.Stream()
out = {}
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e.score_device(dpl.data_ptr(), B, dv.data_ptr(), ds.data_ptr(), True, s.cuda_stream)
    torch.cuda.synchronize()
    out["device_ms"] = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    e.score_best_host_ptr(host.data_ptr(), B, hv.data_ptr(), hs.data_ptr(), True)
    out["host_best_ms"] = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    e.score_best_host_ptr(host.data_ptr(), B, 0, 0, True)
    out["host_best_novals_ms"] = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    dpl.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    out["h2d_ms"] = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    hv.copy_(dv, non_blocking=True)
    hs.copy_(ds, non_blocking=True)
    torch.cuda.synchronize()
    out["d2h_ms"] = (time.perf_counter() - t0) * 1e3
    print(json.dumps(out))
