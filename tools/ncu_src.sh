#!/bin/bash
# Source-level ncu captures (kept as .ncu-rep) of single level-pass launches:
# cfg5 deep levels (multi-segment tiles) and one cfg3 u8 level pass.
set -u
mkdir -p gpurun_out
CMD3="python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-extra --no-graph"
CMD5="python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-extra --no-graph"
$CMD3 > gpurun_out/src_plain3.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:'k_level' -s 20 -c 1 -o gpurun_out/src_cfg3 $CMD3 > gpurun_out/src_ncu3.log 2>&1
echo "rc3=$?" >> gpurun_out/src_ncu3.log
$CMD5 > gpurun_out/src_plain5.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:'k_level' -s 86 -c 1 -o gpurun_out/src_cfg5 $CMD5 > gpurun_out/src_ncu5.log 2>&1
echo "rc5=$?" >> gpurun_out/src_ncu5.log
for c in 3 5; do
  ncu -i gpurun_out/src_cfg$c.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_cfg$c.csv 2>/dev/null
  python tools/ncu_lines.py gpurun_out/src_cfg$c.csv 60 > gpurun_out/src_lines$c.txt 2>&1
done
ls -la gpurun_out
