set -x
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/scale_n1.log 2>&1; echo n1=$?
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus $N > gpurun_out/scale_n$N.log 2>&1; echo n$N=$?
done
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/scale_ref.log 2>&1; echo ref=$?
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --config syn256-120l --per-gpu 200000 --steps 5 --no-routing --no-configs > gpurun_out/syn_n1.log 2>&1; echo s1=$?
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29518 bench.py --config syn256-120l --per-gpu 200000 --steps 5 --gpus $N > gpurun_out/syn_n$N.log 2>&1; echo s$N=$?
done
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --impl reference --config syn256-120l --steps 3 --warmup 3 > gpurun_out/syn_ref.log 2>&1; echo sref=$?
