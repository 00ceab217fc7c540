#!/bin/bash
# Build libyy.so for sm_100a (in-tree).  Usage: build.sh [outdir]
# Translation units compile in parallel; the line-sweep file once per quantity.
set -e
HERE="$(cd "$(dirname "$0")" && pwd)"
OUT="${1:-$HERE/..}"
NVCC="${NVCC:-/usr/local/cuda/bin/nvcc}"
FLAGS="${YY_EXTRA_FLAGS:-} -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v"
OBJ="$(mktemp -d)"
trap 'rm -rf "$OBJ"' EXIT
pids=()
"$NVCC" $FLAGS -c -o "$OBJ/api.o" "$HERE/yy_api.cu" 2> "$OBJ/api.log" & pids+=($!)
"$NVCC" $FLAGS -c -o "$OBJ/kernels.o" "$HERE/yy_kernels.cu" 2> "$OBJ/kernels.log" & pids+=($!)
"$NVCC" $FLAGS -c -o "$OBJ/slab.o" "$HERE/yy_slab.cu" 2> "$OBJ/slab.log" & pids+=($!)
# one wrapper file per quantity: distinct file names give distinct CUDA module
# ids (TUs compiled from the same file name collide at fatbin registration)
for q in 0 1 2 3; do
  printf '#define YY_LINE_Q %d\n#include "%s/yy_line.cu"\n' $q "$HERE" > "$OBJ/yy_line_q$q.cu"
  "$NVCC" $FLAGS -I"$HERE" -c -o "$OBJ/line$q.o" "$OBJ/yy_line_q$q.cu" 2> "$OBJ/line$q.log" & pids+=($!)
done
rc=0
for p in "${pids[@]}"; do wait "$p" || rc=1; done
cat "$OBJ"/*.log > "$OUT/.ptxas.log"
if [ $rc -ne 0 ]; then grep -i -B2 -A3 "error" "$OUT/.ptxas.log" | head -60; exit 1; fi
"$NVCC" -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT/libyy.so" "$OBJ"/*.o
# a host call to a __device__-only function compiles to exit(1) in the host code:
# refuse such a library
if command -v objdump > /dev/null && objdump -d "$OUT/libyy.so" | grep -q "call.*<exit@plt>"; then
  echo "build.sh: libyy.so calls exit() (host code calls a __device__-only function)" >&2
  exit 1
fi
