#!/bin/bash
# Source-level ncu capture of one cfg4 (u16) level pass and the cfg2 pair pass.
set -u
mkdir -p gpurun_out
CMD4="python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-extra --no-graph"
CMD2="python bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-extra --no-graph"
$CMD4 > gpurun_out/src_plain4.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:'k_level' -s 46 -c 1 -o gpurun_out/src_cfg4 $CMD4 > gpurun_out/src_ncu4.log 2>&1
$CMD2 > gpurun_out/src_plain2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:'k_pair2' -s 3 -c 1 -o gpurun_out/src_cfg2 $CMD2 > gpurun_out/src_ncu2.log 2>&1
for c in 4 2; do
  ncu -i gpurun_out/src_cfg$c.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_cfg$c.csv 2>/dev/null
  python tools/ncu_lines.py gpurun_out/src_cfg$c.csv 70 > gpurun_out/src_lines$c.txt 2>&1
  ncu -i gpurun_out/src_cfg$c.ncu-rep --page raw --csv > gpurun_out/src_raw$c.csv 2>/dev/null
  rm -f gpurun_out/src_cfg$c.csv
done
