"""plan(c, method) objective and wall seconds per method and config (one GPU)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json,time,paper_2406_01566_b200 as h
from paper_2406_01566_b200 import clusters
for n in sys.argv[1:] or ("het42-70b","geo24","geo24-70b","single24-70b","syn256-120l"):
    c=h.Cluster.from_json(json.dumps(clusters.CONFIGS[n]()))
    out={"config":n}
    for m in ("swarm","petals","sp","local","sampled"):
        try:
            t=time.time(); p=h.plan(c,m); out[m]=[round(p.objective,2), round(time.time()-t,2)]
        except Exception as e: out[m]=str(e)[:80]
    print(json.dumps(out), flush=True)
