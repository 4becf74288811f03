#!/bin/bash
set -u
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
WT_QUAD=2 WT_DEBUG_SYNC=1 timeout 300 python tools/quad_check.py > gpurun_out/quad_check.log 2>&1; echo "rc=$?" >> gpurun_out/quad_check.log
for c in 3 4 5; do
  WT_QUAD=2 timeout 300 python bench.py --config $c --no-cpu-baseline --no-extra --no-graph --e2e-steps 1 --out gpurun_out/qw_cfg$c.json > gpurun_out/qw_cfg$c.log 2>&1
done
