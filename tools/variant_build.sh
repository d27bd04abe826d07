#!/bin/bash
# Build libks_b200.so with extra nvcc defines into paper_1312_1869_b200/variants/<name>.so (A/B timing on one box).
# usage: tools/variant_build.sh name "-DFOO=1 -DBAR=0"
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p paper_1312_1869_b200/variants /tmp/ksv_$name
for f in ks_api ks_sketch ks_gauss ks_tsqr ks_solve ks_gp; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -Xcompiler -fvisibility=hidden -cudart static $1 -c paper_1312_1869_b200/csrc/$f.cu -o /tmp/ksv_$name/$f.o &
done
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -cudart static -o paper_1312_1869_b200/variants/$name.so /tmp/ksv_$name/*.o
echo built paper_1312_1869_b200/variants/$name.so
