#!/bin/bash
cd $GRAFT_REPO_ROOT
PROBE_SPEC_ONLY=1 timeout 600 python tools/route_spec_probe.py 1000000 > gpurun_out/r02z_spec.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "route or masked" > gpurun_out/r02z_tests.log 2>&1
