#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 compute-sanitizer --print-limit 5 python tools/repro_het42.py > gpurun_out/r02h_sanitizer.log 2>&1
