#!/bin/bash
# A/B timing of an alternative library build against the current one (bench, kernel-only)
python -c 'import __graft_entry__ as g; g.build()' > /dev/null 2>&1
for c in ${CFGS:-4}; do
  for v in cur alt cur alt; do
    if [ $v = cur ]; then unset WT_LIB; else export WT_LIB=$PWD/tools/libwt_alt.so; fi
    timeout 300 python bench.py --config $c --steps 20 --no-cpu-baseline --e2e-steps 0 --out gpurun_out/ab_${v}_cfg$c.json > /dev/null 2>&1
    python tools/summ.py gpurun_out/ab_${v}_cfg$c.json | grep -E "per launch" | cut -c1-120 | sed "s/^/$v cfg$c /" >> gpurun_out/ab.log
  done
done
