"""One scoring launch for ncu: python tools/profile_score.py [--config het42-70b] [--count 200000]."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2406_01566_b200 as h  # noqa: E402
from paper_2406_01566_b200 import clusters  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="het42-70b")
ap.add_argument("--count", type=int, default=200_000)
ap.add_argument("--repeat", type=int, default=1)
ap.add_argument("--mode", default="score", choices=["score", "parity"])
ap.add_argument("--walk", action="store_true", help="link-walking generator (sparse topologies)")
a = ap.parse_args()
c = h.Cluster.from_json(json.dumps(clusters.CONFIGS[a.config]("float")))
e = h.Engine(c)
e.mode = a.mode
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
pl = torch.empty((a.count, e.num_nodes, 2), dtype=torch.int16, device="cuda")
if a.walk:
    e.generate_walk_device(20240611, 0, a.count, pl.data_ptr(), s.cuda_stream)
else:
    e.generate_device(20240611, 0, a.count, 0, pl.data_ptr(), s.cuda_stream)
v = torch.empty(a.count, dtype=torch.float64, device="cuda")
st = torch.empty(a.count, dtype=torch.int32, device="cuda")
for _ in range(a.repeat):
    e.score_device(pl.data_ptr(), a.count, v.data_ptr(), st.data_ptr(), True, s.cuda_stream)
torch.cuda.synchronize()
print(json.dumps({"mode": a.mode, "config": a.config, "count": a.count, "kernel_ms": e.last_kernel_ms(),
                  "evals_per_s": a.count / (e.last_kernel_ms() / 1e3), "mean_value": float(v.mean())}))
