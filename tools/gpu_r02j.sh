#!/bin/bash
cd $GRAFT_REPO_ROOT
for v in p64 p72 lb8 lb7 nat; do
  LP=$PWD/build/var_$v/lib
  echo "== $v" >> gpurun_out/r02j_variants.log
  LD_LIBRARY_PATH=$LP timeout 300 python tools/repro_het42.py >> gpurun_out/r02j_variants.log 2>&1
  LD_LIBRARY_PATH=$LP timeout 300 python tools/profile_score.py --mode parity --count 200000 --repeat 3 >> gpurun_out/r02j_variants.log 2>&1
  LD_LIBRARY_PATH=$LP timeout 300 python tools/profile_score.py --mode score --count 1000000 --repeat 3 >> gpurun_out/r02j_variants.log 2>&1
done
