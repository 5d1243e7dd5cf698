set -x
timeout 900 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_n1.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_n1.log | cut -c1-300
timeout 900 python bench.py --config syn256-120l --per-gpu 200000 --steps 5 --no-routing --no-configs > gpurun_out/syn_n1.log 2>&1; echo s1=$?; tail -1 gpurun_out/syn_n1.log | cut -c1-300
timeout 600 python tools/profile_score.py --config syn256-120l --walk --count 20000 > gpurun_out/syn_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -c 1 -o gpurun_out/r01_syn256_score python tools/profile_score.py --config syn256-120l --walk --count 20000 > gpurun_out/ncu_syn.log 2>&1; echo ncu=$?
