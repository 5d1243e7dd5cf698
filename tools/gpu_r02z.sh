#!/bin/bash
cd $GRAFT_REPO_ROOT
for v in prof_iso; do
HELIO_ROUTE_DIAG=1 LD_LIBRARY_PATH=$PWD/build/var_$v/lib timeout 300 python tools/route_masked_probe.py 1000000 golden 5e6 > gpurun_out/r02z_${v}_gold5.log 2>&1
HELIO_ROUTE_DIAG=1 LD_LIBRARY_PATH=$PWD/build/var_$v/lib timeout 300 python tools/route_masked_probe.py 1000000 bench 1e6 > gpurun_out/r02z_${v}_bench.log 2>&1
done
