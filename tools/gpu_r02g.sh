#!/bin/bash
# round-2: kernel split (per-kernel register budgets) + syn256 ILP: het42 / syn256 lines, parity subset
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_reference_cases.py -m gpu -q -x > gpurun_out/r02g_tests.log 2>&1
echo "exit $?" >> gpurun_out/r02g_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-configs --no-routing --no-cpu-baseline > gpurun_out/r02g_het42.json 2> gpurun_out/r02g_het42.err
timeout 600 python bench.py --config syn256-120l --global-batch 200000 --steps 5 --warmup 3 --no-configs --no-routing --no-cpu-baseline --no-e2e > gpurun_out/r02g_syn256.json 2> gpurun_out/r02g_syn256.err
