#!/bin/bash
cd $GRAFT_REPO_ROOT
HELIO_ROUTE_DIAG=1 LD_LIBRARY_PATH=$PWD/build/var_prof/lib timeout 300 python tools/route_masked_probe.py 1000000 bench 1e6 > gpurun_out/r02z_prof_bench.log 2>&1
