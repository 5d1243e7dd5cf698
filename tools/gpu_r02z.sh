#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02z_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r02z_smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02z_gpu_tests.log 2>&1; echo "exit $?" >> gpurun_out/r02z_gpu_tests.log
timeout 1200 python bench.py > gpurun_out/r02z_bench.json 2> gpurun_out/r02z_bench.err
timeout 1500 python bench.py --config syn256-120l --steps 5 --warmup 3 > gpurun_out/r02z_bench_syn.json 2> gpurun_out/r02z_bench_syn.err
