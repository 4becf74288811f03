#!/bin/bash
# A/B of experiment libraries (tools/libwt_<name>.so, base = in-tree) with tools/ab_cfg.py:
# LIBS="base x" CFGS="3 5" bash tools/ab_quick.sh  -> gpurun_out/ab_quick.log
set -u
mkdir -p gpurun_out
for c in ${CFGS:-3 4 5}; do
  for rep in 1 2; do
    for v in ${LIBS:-base}; do
      if [ $v = base ]; then unset WT_LIB; else export WT_LIB=$PWD/tools/libwt_$v.so; fi
      timeout 300 python tools/ab_cfg.py $c ${REPS:-10} >> gpurun_out/ab_quick.log 2>&1
    done
  done
done
