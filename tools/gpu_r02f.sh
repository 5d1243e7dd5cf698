#!/bin/bash
# round-2 (2 GPUs): multi-GPU tests, masked routing timing + parity
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_multi_gpu.py -m gpu -q > gpurun_out/r02f_multi.log 2>&1
echo "exit $?" >> gpurun_out/r02f_multi.log
python tools/route_masked_probe.py 1000000 > gpurun_out/r02f_masked.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_planner_sim.py -m gpu -q -k "masked or routes or kvmask" > gpurun_out/r02f_tests.log 2>&1
echo "exit $?" >> gpurun_out/r02f_tests.log
