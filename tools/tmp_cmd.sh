#!/bin/bash
set -u
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
for r in 1 2; do
for v in lut1 main lut2 lut8; do
  if [ $v = main ]; then L=""; else L=tools/libwt_$v.so; fi
  echo "== $v" >> gpurun_out/ab_lut.log
  WT_LIB=$L timeout 300 python tools/ab_cfg.py 2 50 >> gpurun_out/ab_lut.log 2>&1
done
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "l2 or config_parity and 2 or edge_sizes" > gpurun_out/pytest_p2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p2.log
