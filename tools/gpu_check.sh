#!/bin/bash
# One GPU session: parity tests, bench per config, launch list.  Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build(); g.smoke()' > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in ${CFGS:-2 3 4 5}; do
  timeout 600 python bench.py --config $c --out gpurun_out/bench_cfg$c.json ${BENCH_ARGS:-} > gpurun_out/bench_cfg$c.log 2>&1; echo "rc=$?" >> gpurun_out/bench_cfg$c.log
done
