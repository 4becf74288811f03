#!/bin/bash
# experiment builds of libwt.so (timing only; results are wrong)
set -e
cd "$(dirname "$0")/.."
for v in NONE SKIP_PCOUNT SKIP_COUNT; do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -cudart shared -Xlinker -rpath,/usr/local/cuda/lib64 -shared -DWT_EXP_$v -DWT_EXP_LEVELS=1 -I include -I paper_1610_05994_b200/csrc -o tools/libwt_$v.so paper_1610_05994_b200/csrc/wt_api.cu &
done
wait
