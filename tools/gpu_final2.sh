# Round-1 final measurements on one 4-GPU box: het42 + syn256 at N = 1/2/4,
# both reference arms (N=1, and torchrun N=2 as the driver launches it), then
# single-GPU ncu captures (het42 SCORE, syn256 SCORE, the bench launch list).
set -x
bash tools/gpu_scale.sh
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29519 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > gpurun_out/scale_ref_n2.log 2>&1; echo ref_n2=$?
bash tools/gpu_syn_scale.sh
export CUDA_VISIBLE_DEVICES=0
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_kernel -c 1 -o gpurun_out/r01_score_final python tools/profile_score.py --mode score > gpurun_out/ncu_s.log 2>&1; echo ncu_het=$?
timeout 600 python tools/profile_score.py --config syn256-120l --walk --count 20000 > gpurun_out/syn_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -c 1 -o gpurun_out/r01_syn256_score python tools/profile_score.py --config syn256-120l --walk --count 20000 > gpurun_out/ncu_syn.log 2>&1; echo ncu_syn=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-routing --no-configs --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
