#!/bin/bash
# Build an A/B variant of libmswm_cuda.so with extra nvcc flags into
# paper_2106_07154_b200/_lib_ab/<name>.so (development tool; load it with
# MSWM_CUDA_LIB=<path> in a separate process).
#   scripts/build_ab.sh <name> [-DMSWM_KOUT_MINB=6 ...]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
mkdir -p "$ROOT/paper_2106_07154_b200/_lib_ab"
/usr/local/cuda/bin/nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false \
  -Xcompiler -fPIC,-ffp-contract=off -Xptxas -v -I"$ROOT/include" "$@" -shared \
  -o "$ROOT/paper_2106_07154_b200/_lib_ab/$name.so" "$ROOT/paper_2106_07154_b200/csrc/mswm_cuda.cu" -lcudart \
  2> "$ROOT/paper_2106_07154_b200/_lib_ab/$name.ptxas.log"
grep -A3 "k_out\|k_vertex_cell" "$ROOT/paper_2106_07154_b200/_lib_ab/$name.ptxas.log" | grep "Used\|spill" | sed 's/ptxas info    : //'
