#!/bin/bash
# tuning sweep of the narrow3d_fast knobs (env) on the configs[1] bench
for pair in 1 0; do for occ in 1 2; do for grid in persistent chunk; do
  SMC_NARROW_PAIR=$pair SMC_NARROW_OCC=$occ SMC_NARROW_GRID=$grid timeout 300 python bench.py --steps 1000 --warmup 20 --no-cpu-baseline --no-ns --no-advance > gpurun_out/b.log 2>&1
  python - "$pair" "$occ" "$grid" <<'PY'
import json, sys
d = json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1])
print('pair=%s occ=%s %s' % tuple(sys.argv[1:4]), round(d['ms_per_step'], 4), round(d['value'] / 1e9, 2),
      round(d['roofline']['frac'], 3), d['clocks']['sm_mhz'])
PY
done; done; done
