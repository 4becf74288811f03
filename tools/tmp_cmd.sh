#!/bin/bash
set -u
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_dd.py tests/test_gpu_dist.py -q -x > gpurun_out/pytest_dd.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dd.log
timeout 600 python bench.py --dd --out gpurun_out/bench_dd1.json > gpurun_out/bench_dd1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_dd1.log
(for c in 3 4 5; do timeout 600 python tools/dd_bench.py $c 2 8; done) > gpurun_out/dd_bench.log 2>&1
