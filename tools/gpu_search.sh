set -x
timeout 900 python -m pytest tests/test_search.py -q -m gpu --timeout 600 > gpurun_out/pytest_search.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_search.log
timeout 900 python bench.py > gpurun_out/bench_n1.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_n1.log | cut -c1-200
