#!/bin/bash
# Quick GPU iteration: a parity subset, then kernel-only bench lines per config.
set -u
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "${PYK:-random_small or edge_sizes or many_tiles or fig2}" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
if grep -q "pytest rc=0" gpurun_out/pytest_quick.log; then
for c in ${CFGS:-3 4 5}; do
  timeout 300 python bench.py --config $c --steps ${STEPS:-20} --no-cpu-baseline --e2e-steps 0 --out gpurun_out/q_cfg$c.json > gpurun_out/q_cfg$c.log 2>&1; echo "rc=$?" >> gpurun_out/q_cfg$c.log
done
fi
