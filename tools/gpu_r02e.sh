#!/bin/bash
# round-2 (2 GPUs): multi-GPU tests, FP64/LDS latency probe, ncu of the masked replay kernel
cd $GRAFT_REPO_ROOT
nvidia-smi -L > gpurun_out/r02e_smi.txt
./tools/micro/lat > gpurun_out/r02e_lat.txt 2>&1
timeout 900 python -m pytest tests/test_multi_gpu.py -m gpu -q > gpurun_out/r02e_multi.log 2>&1
echo "exit $?" >> gpurun_out/r02e_multi.log
timeout 600 ncu --set full --import-source on -k regex:route_masked_warp -c 1 -o gpurun_out/r02e_masked \
  python tools/route_masked_probe.py 200000 > gpurun_out/r02e_ncu.log 2>&1
