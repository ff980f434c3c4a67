#!/bin/bash
# build_ntt_variant.sh NAME "NVCC -D flags": the library with ntt.cu rebuilt under the flags -> build_ab/NAME/libfheon_b200.so
set -e
name=$1; flags=$2
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/build_ab/$name; mkdir -p $out
cd $root/paper_2510_03996_b200/csrc
/usr/local/cuda/bin/nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
  -Xcompiler -fopenmp -Xcompiler -ffp-contract=off --expt-relaxed-constexpr $flags -c ntt.cu -o $out/ntt.o
objs=$(ls ../_lib/obj/*.o | grep -v '/ntt.o')
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fopenmp $objs $out/ntt.o -o $out/libfheon_b200.so -lcudart
echo built $out/libfheon_b200.so
