#!/usr/bin/env bash
# Build libpcsir_b200.so in-tree for sm_100a.
set -euo pipefail
cd "$(dirname "$0")"
OUT=paper_1310_5541_b200/libpcsir_b200.so
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared -Xptxas -v ${PCS_NVCC_EXTRA:-} \
  -o "$OUT" paper_1310_5541_b200/csrc/pcs_capi.cu 2> build_ptxas.log || { cat build_ptxas.log; exit 1; }
echo "built $OUT"
