"""One masked-routing call for ncu: python tools/route_masked_probe.py [requests] [golden|bench] [kv].
golden = the golden geo24 plan (tests/golden/route_geo24.npz); bench = bench.py
routing_leg's plan (first max of 100k geo24 candidates)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
sys.path.insert(0, "tools")
import paper_2406_01566_b200 as h  # noqa: E402
from _support import golden, golden_cluster  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
which = sys.argv[2] if len(sys.argv) > 2 else "golden"
kv = float(sys.argv[3]) if len(sys.argv) > 3 else 1e6
if which == "bench":
    from route_spec_probe import bench_plan  # noqa: E402
    d, row, pe, pf = bench_plan()
else:
    z = golden("route_geo24.npz")
    d = golden_cluster("geo24_float")
    row, pf = z["row"], z["plan_flow"]
    pe = np.stack([z["plan_src"], z["plan_dst"], z["plan_es"], z["plan_ee"]], 1).astype(np.int32)
d = json.loads(json.dumps(d))
d["model"]["kv_bytes_per_token_layer"] = kv
c = h.Cluster.from_json(json.dumps(d))
e = h.Engine(c)
_, inl, outl = h.generate_trace_arrays(R, 0.0, "offline", 7)
for _ in range(2):
    t0 = time.perf_counter()
    nh, hn, hs, he, den = e.route(row, pe, pf, inl, outl, 0, False)
    dt = time.perf_counter() - t0
    print(f"deferred {den}  {R / dt / 1e6:.3f}M routes/s (host wall, incl. copies)")
