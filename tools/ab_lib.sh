#!/bin/bash
# Build libdamf_gpu.so of git revision $1 into paper_2306_08967_b200/libdamf_gpu_ab.so
# (same-box A/B timing: DAMF_GPU_LIB=... selects it).
set -e
rev=${1:-HEAD}
tmp=$(mktemp -d)
git -C "$(dirname "$0")/.." archive "$rev" paper_2306_08967_b200/csrc include | tar -x -C "$tmp"
out=$(cd "$(dirname "$0")/.." && pwd)/paper_2306_08967_b200/libdamf_gpu_ab.so
objs=""
for f in "$tmp"/paper_2306_08967_b200/csrc/*.cu; do
  o="$tmp/$(basename "$f" .cu).o"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
       --expt-relaxed-constexpr -diag-suppress 177,550 -c "$f" -o "$o" &
  objs="$objs $o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$out" $objs
rm -rf "$tmp"
echo "built $out from $rev"
