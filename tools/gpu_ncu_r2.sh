#!/bin/bash
# ncu evidence: per config the launch list of one bench build and one --set full capture of the
# roofline kernel(s).  Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
cap() {  # cfg tag kregex skip count
  local CFG=$1 TAG=$2 K=$3 SKIP=$4 COUNT=$5
  local CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-extra --no-graph"
  $CMD > gpurun_out/plain_$TAG.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg$CFG.csv $CMD > gpurun_out/ncu_launches_$TAG.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:"$K" -s $SKIP -c $COUNT -o gpurun_out/prof_cfg$CFG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
  echo "rc=$?" >> gpurun_out/ncu_full_$TAG.log
}
cap 2 cfg2 'k_pair2$' 3 1
cap 3 cfg3 'k_level' 21 7
cap 4 cfg4 'k_level' 45 15
cap 5 cfg5 'k_level' 69 23
