"""Per-call latency breakdown on het42 (bench.py latency leg's placement):
host p50 of max_flow_value / plan_for_placement / Engine.score on one row, for
ncu's kernel durations of the same calls.  python tools/percall_probe.py [n]"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2406_01566_b200 as h  # noqa: E402
from paper_2406_01566_b200 import clusters  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
d = clusters.CONFIGS["het42-70b"]("float")
c = h.Cluster.from_json(json.dumps(d))
eng = h.Engine(c)
row = h.generate_host(list(eng.kmax), c.num_layers, 20240611, 0, 1, 0)[0]
placement = {c.node_ids[k]: (int(row[k, 0]), int(row[k, 1])) for k in range(len(row)) if row[k, 1] > row[k, 0]}
rows1 = np.ascontiguousarray(row[None], np.int16)


def p50(fn):
    fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)) * 1e6


out = {"max_flow_value_us": p50(lambda: h.max_flow_value(c, placement)),
       "plan_for_placement_us": p50(lambda: h.plan_for_placement(c, placement)),
       "engine_score_parity_us": p50(lambda: eng.score(rows1))}
eng.mode = "score"
out["engine_score_score_us"] = p50(lambda: eng.score(rows1))
print(json.dumps(out))
