#!/bin/bash
cd $GRAFT_REPO_ROOT
for v in bcnat; do echo "== $v"; LD_LIBRARY_PATH=$PWD/build/var_$v/lib timeout 300 python tools/repro_het42.py 2>&1 | head -4; done > gpurun_out/r02s_diag.log 2>&1
