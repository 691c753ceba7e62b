#!/bin/bash
# quick per-config timing (no CPU baseline); usage: quick_bench.sh "4 3" [refill_min]
CFGS=${1:-"4"}
R=${2:-4}
for c in $CFGS; do
  timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $c --refill-min $R > gpurun_out/qb_$c.log 2>&1
  tail -1 gpurun_out/qb_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg%s'%$c, 'ms', round(d['ms_per_step'],4), 'Gsteps/s', round(d['value']/1e9,2), d['roofline']['bound'], 'frac', round(d['roofline']['frac'],4))" || tail -4 gpurun_out/qb_$c.log
done
