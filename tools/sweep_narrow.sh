#!/bin/bash
# tuning sweep of the narrow3d_fast knobs (env) on the configs[1] bench
for grid in chunk persistent; do for unr in 0; do for kc in 0 16 24 32; do
  [ "$grid" = persistent ] && [ "$kc" != 0 ] && continue
  SMC_NARROW_GRID=$grid SMC_NARROW_UNROLL=$unr timeout 300 python bench.py --steps 1000 --warmup 20 --no-cpu-baseline --kc $kc > gpurun_out/b.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]);print('$grid unroll=$unr kc=$kc', round(d['ms_per_step'],4), round(d['value']/1e9,2), round(d['roofline']['frac'],3))"
done; done; done
