"""One masked-routing call (geo24 plan, kv_bytes_per_token_layer = 1e6, 1M
requests) for ncu: python tools/route_masked_probe.py [requests]."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2406_01566_b200 as h  # noqa: E402
from _support import golden, golden_cluster  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
z = golden("route_geo24.npz")
d = golden_cluster("geo24_float")
d["model"]["kv_bytes_per_token_layer"] = 1e6
c = h.Cluster.from_json(json.dumps(d))
e = h.Engine(c)
_, inl, outl = h.generate_trace_arrays(R, 0.0, "offline", 7)
pe = np.stack([z["plan_src"], z["plan_dst"], z["plan_es"], z["plan_ee"]], 1).astype(np.int32)
import time  # noqa: E402
for _ in range(3):
    t0 = time.perf_counter()
    nh, hn, hs, he, den = e.route(z["row"], pe, z["plan_flow"], inl, outl, 0, False)
    dt = time.perf_counter() - t0
    print(f"deferred {den}  {R / dt / 1e6:.3f}M routes/s (host wall, incl. copies)")
