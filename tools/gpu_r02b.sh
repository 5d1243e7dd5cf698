#!/bin/bash
# round-2: new planner/scheduler tests + the full GPU suite
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_planner_sim.py -m gpu -q -x > gpurun_out/r02b_planner.log 2>&1
echo "exit $?" >> gpurun_out/r02b_planner.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02b_gpu_tests.log 2>&1
echo "exit $?" >> gpurun_out/r02b_gpu_tests.log
