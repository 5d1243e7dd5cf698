#!/bin/bash
cd $GRAFT_REPO_ROOT
for v in bcnat bc8 nb8; do echo "== $v"; LD_LIBRARY_PATH=$PWD/build/var_$v/lib timeout 300 python tools/repro_het42.py 2>&1 | head -4; LD_LIBRARY_PATH=$PWD/build/var_$v/lib timeout 300 python tools/profile_score.py --mode parity --count 200000 --repeat 2 2>&1 | tail -1; done > gpurun_out/r02t_diag.log 2>&1
echo "== production" >> gpurun_out/r02t_diag.log
timeout 300 python tools/profile_score.py --mode parity --count 200000 --repeat 3 >> gpurun_out/r02t_diag.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02t_gpu_tests.log 2>&1
echo "exit $?" >> gpurun_out/r02t_gpu_tests.log
