#!/bin/bash
# cfg1 as one estimate (latency) and as 2/4/8/16 replicas per launch
for R in 1 2 4 8 16; do
  python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline --no-extras --replicas $R 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg1 x$R ms', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4))"
done
