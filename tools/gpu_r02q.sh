#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_planner_sim.py -m gpu -q -k "masked or routes or kvmask or simulate" > gpurun_out/r02q_tests.log 2>&1
echo "exit $?" >> gpurun_out/r02q_tests.log
timeout 600 python - > gpurun_out/r02q_routing.json 2> gpurun_out/r02q_routing.err <<'PY'
import json, sys, torch
sys.path.insert(0, ".")
import bench
import paper_2406_01566_b200 as h
from paper_2406_01566_b200 import clusters
s = torch.cuda.Stream()
print(json.dumps(bench.routing_leg(h, clusters, 0, s.cuda_stream, 1_000_000, True)))
PY
python tools/route_masked_probe.py 1000000 > gpurun_out/r02q_masked.txt 2>&1
for v in nb8 bc8; do echo "== $v"; LD_LIBRARY_PATH=$PWD/build/var_$v/lib timeout 300 python tools/repro_het42.py 2>&1 | tail -5; done > gpurun_out/r02q_diag.log 2>&1
