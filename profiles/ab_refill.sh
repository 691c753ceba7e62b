#!/bin/bash
# cfg4 time against the hot loop's refill threshold (runtime tuning, no rebuild)
for r in "$@"; do
  timeout 120 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras --refill-min $r > gpurun_out/rf_$r.log 2>&1
  tail -1 gpurun_out/rf_$r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('refill_min $r', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4))" || tail -3 gpurun_out/rf_$r.log
done
