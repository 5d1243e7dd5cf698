#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02k_gpu_tests.log 2>&1
echo "exit $?" >> gpurun_out/r02k_gpu_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-configs --no-routing --no-cpu-baseline > gpurun_out/r02k_het42.json 2> gpurun_out/r02k_het42.err
timeout 600 python bench.py --config syn256-120l --global-batch 200000 --steps 5 --warmup 3 --no-configs --no-routing --no-cpu-baseline --no-e2e > gpurun_out/r02k_syn256.json 2> gpurun_out/r02k_syn256.err
