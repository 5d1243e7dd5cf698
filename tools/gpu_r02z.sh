#!/bin/bash
cd $GRAFT_REPO_ROOT
for i in 1 2; do timeout 300 python tools/profile_score.py --config syn256-120l --walk --count 200000 --repeat 3; done > gpurun_out/r02z_syn.log 2>&1
timeout 900 python tools/syn256_determinism.py 10000000 > gpurun_out/r02z_det.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_search.py -m gpu -q -k "syn256 or push_relabel or size_sweep or walk or dense or tiny or beyond or prune or mesh or global" > gpurun_out/r02z_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02z_tests.log
timeout 900 python tools/fuzz_parity.py --seconds 240 --seed 21 > gpurun_out/r02z_fuzz.log 2>&1; echo "exit $?" >> gpurun_out/r02z_fuzz.log
