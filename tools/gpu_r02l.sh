#!/bin/bash
# ncu --set full of the dominant score_kernel launch: syn256 (large-graph SCORE kernel) and het42 SCORE
cd $GRAFT_REPO_ROOT
timeout 300 python tools/profile_score.py --config syn256-120l --walk --count 20000 > gpurun_out/r02l_syn_plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -c 1 -o gpurun_out/r02l_syn256 python tools/profile_score.py --config syn256-120l --walk --count 20000 > gpurun_out/r02l_ncu_syn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -c 1 -o gpurun_out/r02l_het42 python tools/profile_score.py --config het42-70b --count 200000 > gpurun_out/r02l_ncu_het42.log 2>&1
