#!/bin/bash
set -u
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_quad.py tests/test_gpu_dist.py -q -x > gpurun_out/pytest_quad.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quad.log
