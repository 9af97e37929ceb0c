#!/bin/bash
# Build the working tree's CUDA sources with extra nvcc flags into
# paper_2306_08967_b200/libdamf_gpu_$1.so (select with DAMF_GPU_LIB=...):
#   tools/build_variant.sh prof -DDAMF_PROF=1
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$root/build/variant_$name
mkdir -p "$tmp"
objs=""
for f in "$root"/paper_2306_08967_b200/csrc/*.cu; do
  o="$tmp/$(basename "$f" .cu).o"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
       --expt-relaxed-constexpr -diag-suppress 177,550 -I"$root/include" "$@" -c "$f" -o "$o" &
  objs="$objs $o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$root/paper_2306_08967_b200/libdamf_gpu_$name.so" $objs
echo "built libdamf_gpu_$name.so"
