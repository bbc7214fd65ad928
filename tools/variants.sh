#!/bin/bash
# Build variant libraries of librt_b200.so with extra nvcc defines into gpurun-travelling dirs:
#   tools/variants.sh NAME "-DFOO=1 -DBAR=2" [NAME "-D..."]...
# -> variants/NAME/librt_b200.so ; use with RT_B200_LIB=variants/NAME/librt_b200.so
set -e
cd "$(dirname "$0")/.."
CS=paper_2603_00292_b200/csrc
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr"
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  out=variants/$name; mkdir -p $out
  pids=()
  for f in capi mesh lbvh trace render tlas multi; do
    /usr/local/cuda/bin/nvcc $FLAGS $defs -c $CS/$f.cu -o $out/$f.o & pids+=($!)
  done
  for p in "${pids[@]}"; do wait $p; done
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/librt_b200.so $out/*.o -lcudart -ldl
  rm -f $out/*.o
  echo "built $out"
done
