#!/bin/bash
# round-2 check: GPU tests, default bench line, reference arm
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02a_gpu_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/r02a_gpu_tests.log
timeout 900 python bench.py > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02a_bench_ref.json 2> gpurun_out/r02a_bench_ref.err
