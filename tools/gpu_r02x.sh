#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_multi_gpu.py tests/test_search.py -m gpu -q > gpurun_out/r02x_tests.log 2>&1
echo "exit $?" >> gpurun_out/r02x_tests.log
