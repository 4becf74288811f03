#!/bin/bash
# Round-end evidence: smoke, the GPU tests, the default bench line, the reference
# arm, the dd step at N = 1, ncu launch lists + captures summarised on the box.
set -u
TAG=${TAG:-r02_v11}
mkdir -p gpurun_out/profiles_out
python -c 'import __graft_entry__ as g; g.build(); g.smoke()' > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1200 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --out gpurun_out/bench_default.json > gpurun_out/bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/bench_default.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference.log 2>&1; echo "rc=$?" >> gpurun_out/bench_reference.log
timeout 600 python bench.py --dd --out gpurun_out/bench_dd1.json > gpurun_out/bench_dd1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_dd1.log
TAG=$TAG bash tools/gpu_ncu_r2.sh > gpurun_out/ncu_all.log 2>&1
du -sh gpurun_out
