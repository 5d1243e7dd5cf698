#!/bin/bash
# Round-2 scaling on one 4-GPU box: het42 strong scaling (1M global) at N = 1, 2, 4 with the
# weak-scaling line beside it, the reference arm under torchrun, syn256 10M at N = 1, 2, 4,
# and the multi-GPU library tests.
cd $GRAFT_REPO_ROOT
O=gpurun_out/scale
mkdir -p $O
nvidia-smi -L > $O/smi.txt
run() {  # n, tag, extra args
  if [ $1 = 1 ]; then
    timeout 900 python bench.py ${@:3} > $O/$2.json 2> $O/$2.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 \
      --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $1 ${@:3} > $O/$2.json 2> $O/$2.err
  fi
}
for n in 1 2 4; do run $n het42_n$n --no-configs --no-routing --no-cpu-baseline; done
run 2 reference_n2 --impl reference
for n in 1 2 4; do run $n syn256_n$n --config syn256-120l --steps 5 --warmup 3 --no-configs --no-routing --no-cpu-baseline; done
timeout 900 python -m pytest tests/test_multi_gpu.py tests/test_dist_gloo.py -q > $O/multi_tests.log 2>&1
echo "exit $?" >> $O/multi_tests.log
