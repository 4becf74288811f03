#!/bin/bash
# A/B of experiment builds (WT_LIB) on bench configs: LIBS="name ..." (tools/libwt_<name>.so; base = in-tree)
set -u
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > /dev/null 2>&1
for v in ${LIBS:-base}; do
  if [ $v = base ]; then unset WT_LIB; else export WT_LIB=$PWD/tools/libwt_$v.so; fi
  if [ -n "${PYK:-}" ]; then timeout 900 python -m pytest tests -m gpu -q -x -k "$PYK" > gpurun_out/ab_pytest_$v.log 2>&1; echo "rc=$?" >> gpurun_out/ab_pytest_$v.log; fi
  for c in ${CFGS:-2}; do
    timeout 300 python bench.py --config $c --steps ${STEPS:-50} --no-cpu-baseline --e2e-steps 0 --no-extra --out gpurun_out/ab_${v}_cfg$c.json > gpurun_out/ab_${v}_cfg$c.log 2>&1
  done
done
