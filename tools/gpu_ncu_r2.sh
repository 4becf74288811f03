#!/bin/bash
# ncu evidence: per config the launch list of one bench build and one --set full capture of the
# roofline kernel(s), summarised ON THE BOX (tools/ncu_summary.py) into gpurun_out/profiles_out/
# (the .ncu-rep files of the multi-kernel captures are too large to bring back).
set -u
TAG=${TAG:-r02_v11}
mkdir -p gpurun_out/profiles_out
cap() {  # cfg kregex skip count keep_rep
  local CFG=$1 K=$2 SKIP=$3 COUNT=$4 KEEP=$5
  local CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-extra --no-graph"
  $CMD > gpurun_out/plain_cfg$CFG.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg$CFG.csv $CMD > gpurun_out/ncu_launches_cfg$CFG.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:"$K" -s $SKIP -c $COUNT -o gpurun_out/prof_cfg$CFG $CMD > gpurun_out/ncu_full_cfg$CFG.log 2>&1
  echo "rc=$?" >> gpurun_out/ncu_full_cfg$CFG.log
  python tools/ncu_summary.py $CFG $TAG >> gpurun_out/ncu_full_cfg$CFG.log 2>&1
  cp profiles/$TAG/ncu_summary_cfg$CFG.txt profiles/ncu_traffic_cfg$CFG.json gpurun_out/profiles_out/ 2>/dev/null
  cp gpurun_out/launches_cfg$CFG.csv gpurun_out/profiles_out/ 2>/dev/null
  [ "$KEEP" = 1 ] || rm -f gpurun_out/prof_cfg$CFG.ncu-rep
}
cap 2 'k_pair2$' 3 1 1
cap 3 'k_level|k_pairn' 21 7 0
cap 4 'k_level|k_pairn' 45 15 0
cap 5 'k_level|k_pairn' 69 23 0
du -sh gpurun_out
