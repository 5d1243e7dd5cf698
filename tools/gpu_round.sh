set -x
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-routing > gpurun_out/bench_full.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_full.log | cut -c1-250; grep -o '"other_mode": {[^}]*}' gpurun_out/bench_full.log; grep -o '"e2e": {[^}]*}' gpurun_out/bench_full.log | cut -c1-120
timeout 300 python tools/profile_score.py --mode score > gpurun_out/prof_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -c 1 -o gpurun_out/prof_score_pair python tools/profile_score.py --mode score > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
