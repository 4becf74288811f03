#!/bin/bash
# A/B timing of the current library with and without an environment switch (default WT_NO_PDL=1)
python -c 'import __graft_entry__ as g; g.build()' > /dev/null 2>&1
SW=${SW:-WT_NO_PDL=1}
for c in ${CFGS:-3}; do
  for v in cur alt cur alt; do
    if [ $v = cur ]; then envs=""; else envs="$SW"; fi
    env $envs timeout 300 python bench.py --config $c --steps 20 --no-cpu-baseline --e2e-steps 0 --out gpurun_out/ab_${v}_cfg$c.json > /dev/null 2>&1
    python tools/summ.py gpurun_out/ab_${v}_cfg$c.json 2>/dev/null | head -1 | sed "s/^/$v /" >> gpurun_out/ab.log
  done
done
