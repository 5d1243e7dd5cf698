#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python tools/profile_score.py --mode parity --count 200000 --repeat 3 > gpurun_out/r02v.log 2>&1
python tools/route_masked_probe.py 1000000 >> gpurun_out/r02v.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_planner_sim.py tests/test_reference_cases.py -m gpu -q -k "masked or routes or kvmask or simulate or division or candidate or raw or scheduler" > gpurun_out/r02v_tests.log 2>&1
echo "exit $?" >> gpurun_out/r02v_tests.log
timeout 600 python - > gpurun_out/r02v_routing.json 2> gpurun_out/r02v_routing.err <<'PY'
import json, sys, torch
sys.path.insert(0, ".")
import bench
import paper_2406_01566_b200 as h
from paper_2406_01566_b200 import clusters
s = torch.cuda.Stream()
print(json.dumps(bench.routing_leg(h, clusters, 0, s.cuda_stream, 1_000_000, True)))
PY
