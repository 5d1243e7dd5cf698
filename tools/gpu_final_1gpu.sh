#!/bin/bash
# Round-2 measurements on one B200: smoke, the GPU suite, the default bench line
# (het42, every leg), the reference arm, the syn256 10M line, launch list.
cd $GRAFT_REPO_ROOT
O=gpurun_out/final1
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt
lscpu | head -20 > $O/lscpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "exit $?" >> $O/gpu_tests.log
timeout 1200 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 1500 python bench.py --config syn256-120l --steps 5 --warmup 3 > $O/bench_syn256_n1.json 2> $O/bench_syn256_n1.err
timeout 900 python bench.py --impl reference --config syn256-120l --steps 5 --warmup 3 > $O/bench_syn256_reference.json 2> $O/bench_syn256_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-configs --no-routing --no-cpu-baseline > $O/ncu_bench.log 2>&1
# the masked routing kernel: one route_masked_spec launch on bench.py's plan (kv 1e6, 200k requests)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:route_masked_spec -c 1 -o $O/masked_spec \
  python tools/route_masked_probe.py 200000 bench 1e6 > $O/ncu_masked.log 2>&1
PROBE_SPEC_ONLY=1 timeout 600 python tools/route_spec_probe.py 1000000 > $O/masked_probe.log 2>&1
