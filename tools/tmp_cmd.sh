#!/bin/bash
set -u
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build(); g.smoke()' > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "l2 or config_parity and 2 or random_small or edge_sizes or two_hundred or range" > gpurun_out/pytest_p2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p2.log
timeout 600 python bench.py --no-extra --no-cpu-baseline --out gpurun_out/bench_p2.json > gpurun_out/bench_p2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_p2.log
