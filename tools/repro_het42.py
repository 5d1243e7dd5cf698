import sys, json
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
import paper_2406_01566_b200 as h
from _support import golden, golden_cluster
for key in ["het42-70b_float"]:
    z = golden(f"cand_{key}.npz")
    c = h.Cluster.from_json(json.dumps(golden_cluster(key)))
    e = h.Engine(c)
    for mode in ["score", "parity"]:
        e.mode = mode
        try:
            v, s = e.score(z["rows"][:64], True)
            print(key, mode, "ok", v[:3])
        except Exception as ex:
            print(key, mode, "FAIL", ex)
            break
