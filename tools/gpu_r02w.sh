#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02w_gpu_tests.log 2>&1
echo "exit $?" >> gpurun_out/r02w_gpu_tests.log
timeout 600 python tools/fuzz_parity.py --seconds 300 --seed 11 > gpurun_out/r02w_fuzz.log 2>&1
echo "exit $?" >> gpurun_out/r02w_fuzz.log
