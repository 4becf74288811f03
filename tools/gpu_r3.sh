#!/bin/bash
# GPU tests + single-launch ncu captures (kept): cfg2 final scan, cfg3 / cfg5 k_pairn
set -u
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
cap() {  # cfg kregex skip tag
  local CMD="python bench.py --config $1 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-extra --no-graph"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$2" -s $3 -c 1 -o gpurun_out/cap_$4 $CMD > gpurun_out/cap_$4.log 2>&1
  echo "rc=$?" >> gpurun_out/cap_$4.log
  ncu -i gpurun_out/cap_$4.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/cap_$4_src.csv 2>/dev/null
  ncu -i gpurun_out/cap_$4.ncu-rep --page raw --csv > gpurun_out/cap_$4_raw.csv 2>/dev/null
}
cap 2 'OpBitsPop' 3 fscan2
cap 5 'k_pairn' 3 pairn5
cap 3 'k_pairn' 3 pairn3
ls -la gpurun_out
