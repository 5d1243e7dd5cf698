set -x
timeout 300 python tools/profile_score.py --config syn256-120l --walk --count 20000 > gpurun_out/syn_prof_plain.log 2>&1; echo plain=$?; cat gpurun_out/syn_prof_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -c 1 -o gpurun_out/syn256_score python tools/profile_score.py --config syn256-120l --walk --count 20000 > gpurun_out/ncu_syn.log 2>&1; echo ncu=$?
