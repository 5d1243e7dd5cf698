#!/bin/bash
# round-2: masked routing v2 parity + timing, latency leg
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_planner_sim.py -m gpu -q -x -k "masked or routes or scheduler or simulate or to_dot" > gpurun_out/r02d_tests.log 2>&1
echo "exit $?" >> gpurun_out/r02d_tests.log
timeout 900 python - > gpurun_out/r02d_legs.json 2> gpurun_out/r02d_legs.err <<'PY'
import json, sys, torch
sys.path.insert(0, ".")
import bench
import paper_2406_01566_b200 as h
from paper_2406_01566_b200 import clusters
s = torch.cuda.Stream()
out = {"routing": bench.routing_leg(h, clusters, 0, s.cuda_stream, 1_000_000, True),
       "latency": bench.latency_leg(h, clusters, True)}
print(json.dumps(out))
PY
