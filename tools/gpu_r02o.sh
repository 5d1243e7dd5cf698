#!/bin/bash
cd $GRAFT_REPO_ROOT
for gr in 10 14 20 28 40; do echo "gr=$gr $(HELIO_PR_GR=$gr timeout 300 python tools/profile_score.py --config syn256-120l --walk --count 200000 --repeat 2)"; done > gpurun_out/r02o_gr.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -c 1 -o gpurun_out/r02o_syn256 python tools/profile_score.py --config syn256-120l --walk --count 20000 > gpurun_out/r02o_ncu.log 2>&1
