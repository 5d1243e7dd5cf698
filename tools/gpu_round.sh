set -x
timeout 900 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-routing --no-configs --no-cpu-baseline > gpurun_out/bench_full.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_full.log | cut -c1-150; grep -o '"other_mode": {[^}]*}' gpurun_out/bench_full.log
