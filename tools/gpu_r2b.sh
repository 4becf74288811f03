#!/bin/bash
# Round-2 (session 2): GPU tests, then ncu captures of single kernels (kept as .ncu-rep).
set -u
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build(); g.smoke()' > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
if [ "${TESTS:-1}" = 1 ]; then
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -k "${PYK:-}" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
capk() {  # cfg kregex skip tag
  local CFG=$1 K=$2 SKIP=$3 TAG=$4
  local CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-extra --no-graph"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $SKIP -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
  echo "rc=$?" >> gpurun_out/ncu_$TAG.log
}
for spec in ${CAPS:-}; do
  IFS=, read -r c k s t <<< "$spec"
  capk $c "$k" $s $t
done
du -sh gpurun_out
