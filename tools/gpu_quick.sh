# quick A/B: SCORE/PARITY kernel rates on het42 and syn256, then the GPU parity + search tests
set -x
timeout 300 python tools/profile_score.py --count 200000 --repeat 3 2>&1 | tail -1
timeout 300 python tools/profile_score.py --config syn256-120l --walk --count 20000 --repeat 2 2>&1 | tail -1
timeout 300 python tools/profile_score.py --count 200000 --repeat 2 --mode parity 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_search.py -q -m gpu --timeout 600 -x > gpurun_out/pytest_parity.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_parity.log
timeout 300 python tools/search_probe.py het42-70b 2>&1 | head -1
