#!/bin/bash
cd $GRAFT_REPO_ROOT
for v in bc8 bcnat; do echo "== $v"; LD_LIBRARY_PATH=$PWD/build/var_$v/lib timeout 300 python tools/repro_het42.py 2>&1 | tail -6; done > gpurun_out/r02r_diag.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:route_masked -c 1 -o gpurun_out/r02r_masked python tools/route_masked_probe.py 200000 > gpurun_out/r02r_ncu.log 2>&1
