#!/bin/bash
# round-2: planner/sim tests, masked routing parity + timing
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_planner_sim.py tests/test_gpu_parity.py -m gpu -q -x -k "simulate or masked or routes or scheduler or milp or plan_edges or to_dot or iwrr" > gpurun_out/r02c_tests.log 2>&1
echo "exit $?" >> gpurun_out/r02c_tests.log
timeout 600 python - > gpurun_out/r02c_routing.json 2> gpurun_out/r02c_routing.err <<'PY'
import json, sys, torch
sys.path.insert(0, ".")
import bench
import paper_2406_01566_b200 as h
from paper_2406_01566_b200 import clusters
s = torch.cuda.Stream()
print(json.dumps(bench.routing_leg(h, clusters, 0, s.cuda_stream, 1_000_000, True)))
PY
