set -x
timeout 300 python tools/profile_score.py --mode parity > gpurun_out/prof_parity_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -c 1 -o gpurun_out/r01_parity_v2 python tools/profile_score.py --mode parity > gpurun_out/ncu_p.log 2>&1; echo ncu_p=$?
