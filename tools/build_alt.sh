#!/bin/bash
# Build tools/libwt_alt.so from the current sources with extra nvcc flags (A/B experiments).
# Usage: bash tools/build_alt.sh -DWT_EXP_SOMETHING
set -e
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
  --expt-relaxed-constexpr -cudart shared -Xlinker -rpath,/usr/local/cuda/lib64 -shared -I include \
  -I paper_1610_05994_b200/csrc "$@" -o tools/libwt_alt.so paper_1610_05994_b200/csrc/wt_api.cu
