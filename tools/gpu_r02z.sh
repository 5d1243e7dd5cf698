#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python tools/fuzz_routing.py --seconds 420 --seed 3 > gpurun_out/r02z_fuzz_routing.log 2>&1
echo "exit $?" >> gpurun_out/r02z_fuzz_routing.log
