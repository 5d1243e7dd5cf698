#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -c 1 -o gpurun_out/r02p_syn256 python tools/profile_score.py --config syn256-120l --walk --count 20000 > gpurun_out/r02p_ncu.log 2>&1
