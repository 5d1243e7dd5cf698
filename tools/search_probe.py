"""Placement-search probe: heuristic seed -> local search -> sampled multi-node search -> local search."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_01566_b200 as h
from paper_2406_01566_b200 import clusters

for name in sys.argv[1:] or ["het42-70b"]:
    d = clusters.CONFIGS[name]()
    c = h.Cluster.from_json(json.dumps(d))
    e = h.Engine(c)
    e.mode = "score"
    for m in ("petals", "swarm"):
        seed = h.placement_rows(c, [h.heuristic_placement(c, m)[0]])[0]
        v0 = e.score(seed[None])[0][0]
        v1, r1, mv, sc = e.local_search(seed)
        for changes in (2, 3, 4):
            t = time.time()
            v2, r2, imp, sc2 = e.sampled_search(r1, True, 30, 1 << 20, changes, 7)
            t2 = time.time() - t
            v3, r3, mv3, sc3 = e.local_search(r2)
            print(json.dumps({"config": name, "seed": m, "seed_value": v0, "ls": v1, "changes": changes,
                              "sampled": v2, "improving_rounds": imp, "scored": sc2, "seconds": round(t2, 3),
                              "ls_after": v3}))
