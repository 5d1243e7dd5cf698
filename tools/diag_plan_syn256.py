import os, sys, json, time
sys.path.insert(0, os.getcwd())
import paper_2406_01566_b200 as h
from paper_2406_01566_b200 import clusters
c = h.Cluster.from_json(json.dumps(clusters.CONFIGS["syn256-120l"]()))
def T(label, f):
    t = time.time(); r = f(); print(label, round(time.time() - t, 2), flush=True); return r
pl = T("heur petals", lambda: h.heuristic_placement(c, "petals")[0])
T("max_flow_value petals", lambda: h.max_flow_value(c, pl))
T("plan petals", lambda: h.plan(c, "petals").objective)
T("local_search petals", lambda: h.local_search(c, pl)[1])
T("plan local", lambda: h.plan(c, "local").objective)
T("plan sampled", lambda: h.plan(c, "sampled").objective)
