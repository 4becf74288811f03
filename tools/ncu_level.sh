#!/bin/bash
# Launch list (all kernels, device time) + one full ncu capture of the level pass.
# Usage: CFG=3 KREGEX=k_level SKIP=3 COUNT=1 bash tools/ncu_level.sh
set -u
CFG=${CFG:-3}; KREGEX=${KREGEX:-k_level}; SKIP=${SKIP:-3}; COUNT=${COUNT:-1}; TAG=${TAG:-cfg$CFG}
mkdir -p gpurun_out
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/plain_$TAG.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launches_$TAG.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s $SKIP -c $COUNT -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full_$TAG.log
