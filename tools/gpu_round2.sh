set -x
timeout 300 python tools/profile_score.py --mode score > gpurun_out/prof_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -c 1 -o gpurun_out/r01_score_v5 python tools/profile_score.py --mode score > gpurun_out/ncu_s.log 2>&1; echo ncu_s=$?
