#!/bin/bash
set -u
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
CMD="python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-extra --no-graph"
# level 20 of the 5th build (22 level launches per build: skip 4 builds + 20)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_level' -s 108 -c 1 -o gpurun_out/lvl5 $CMD > gpurun_out/ncu_lvl5.log 2>&1
echo rc=$? >> gpurun_out/ncu_lvl5.log
