#!/bin/bash
cd $GRAFT_REPO_ROOT
for v in default p255 s255; do
  if [ $v = default ]; then LP=""; else LP=$PWD/build/var_$v/lib; fi
  echo "== $v" >> gpurun_out/r02i_bisect.log
  LD_LIBRARY_PATH=$LP timeout 300 python tools/repro_het42.py >> gpurun_out/r02i_bisect.log 2>&1
done
