#!/bin/bash
# build a variant libhelio_gpu.so into build/var_$1 with extra nvcc flags $2
set -e
cd /root/repo
mkdir -p build/var_$1/obj build/var_$1/lib
for f in helio_gpu route search split multi; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC --expt-relaxed-constexpr $2 -c paper_2406_01566_b200/csrc/$f.cu -o build/var_$1/obj/$f.o
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/var_$1/lib/libhelio_gpu.so build/var_$1/obj/*.o -lcudart_static -ldl
