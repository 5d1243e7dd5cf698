set -x
export CUDA_VISIBLE_DEVICES=0
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/profile_score.py --config syn256-120l --walk --count 300 > gpurun_out/san_mem_syn.log 2>&1; echo mem_syn=$?; tail -4 gpurun_out/san_mem_syn.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/profile_score.py --config syn256-120l --walk --count 100 > gpurun_out/san_race_syn.log 2>&1; echo race_syn=$?; tail -4 gpurun_out/san_race_syn.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/profile_score.py --count 3000 > gpurun_out/san_mem_het.log 2>&1; echo mem_het=$?; tail -4 gpurun_out/san_mem_het.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/profile_score.py --count 300 > gpurun_out/san_race_het.log 2>&1; echo race_het=$?; tail -4 gpurun_out/san_race_het.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/profile_score.py --config syn256-120l --walk --count 300 > gpurun_out/san_sync_syn.log 2>&1; echo sync_syn=$?; tail -4 gpurun_out/san_sync_syn.log
