#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_search.py -m gpu -q -x -k "syn256 or push_relabel or size_sweep or walk or dense or tiny or beyond or prune" > gpurun_out/r02n_tests.log 2>&1
echo "exit $?" >> gpurun_out/r02n_tests.log
for i in 1 2; do timeout 300 python tools/profile_score.py --config syn256-120l --walk --count 200000 --repeat 3; done > gpurun_out/r02n_syn.log 2>&1
