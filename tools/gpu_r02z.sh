#!/bin/bash
cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
timeout 900 python bench.py --config syn256-120l --steps 5 --warmup 3 --no-configs --no-routing --no-cpu-baseline > gpurun_out/r02z_syn_$i.json 2> gpurun_out/r02z_syn_$i.err
done
timeout 900 python bench.py --steps 10 --warmup 3 --no-configs --no-routing --no-cpu-baseline > gpurun_out/r02z_het.json 2> gpurun_out/r02z_het.err
