#!/bin/bash
# time the level pass of experiment builds (cfg 3), results are not checked
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > /dev/null 2>&1
for v in NONE SKIP_PCOUNT SKIP_COUNT; do
  if [ $v = base ]; then unset WT_LIB; else export WT_LIB=$PWD/tools/libwt_$v.so; fi
  for c in ${CFGS:-3}; do
    timeout 300 python bench.py --config $c --steps 20 --no-cpu-baseline --e2e-steps 0 --out gpurun_out/exp_${v}_cfg$c.json > gpurun_out/exp_${v}_cfg$c.log 2>&1
  done
done
