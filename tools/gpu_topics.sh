#!/bin/bash
# Topic benches (NEXT rows) with the current kernels: locality sweep, wavelet
# matrix, select index, dd merge.
set -u
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > /dev/null 2>&1
timeout 900 python tools/locality_sweep.py --out gpurun_out/locality_sweep.json > gpurun_out/locality_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/locality_sweep.log
timeout 600 python tools/matrix_bench.py > gpurun_out/matrix_bench.log 2>&1; echo "rc=$?" >> gpurun_out/matrix_bench.log
for c in 3 5; do timeout 600 python tools/select_bench.py $c >> gpurun_out/select_bench.log 2>&1; echo "rc=$?" >> gpurun_out/select_bench.log; done
for c in 3 4 5; do timeout 900 python tools/dd_bench.py $c 2 8 >> gpurun_out/dd_bench.log 2>&1; echo "rc=$?" >> gpurun_out/dd_bench.log; done
