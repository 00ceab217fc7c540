#!/bin/bash
# Build libyy.so for sm_100a (in-tree).  Usage: build.sh [outdir]
set -e
HERE="$(cd "$(dirname "$0")" && pwd)"
OUT="${1:-$HERE/..}"
NVCC="${NVCC:-/usr/local/cuda/bin/nvcc}"
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -Xptxas -v"
"$NVCC" $FLAGS -o "$OUT/libyy.so" "$HERE/yy_api.cu" "$HERE/yy_kernels.cu" 2> "$OUT/.ptxas.log" || { cat "$OUT/.ptxas.log"; exit 1; }
