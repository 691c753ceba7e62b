#!/bin/bash
# quick per-config timing (no CPU baseline); usage: quick_bench.sh "4 3" [refill_min] [refill_min_deferred]
# small configs run with label replicas per launch (cfg0 x64, cfg1 x16, cfg2 x16)
CFGS=${1:-"4"}
R=${2:-5}
RD=${3:-12}
for c in $CFGS; do
  case $c in 0) REP=64;; 1) REP=16;; 2) REP=16;; *) REP=1;; esac
  timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $c --replicas $REP --refill-min $R --refill-min-deferred $RD > gpurun_out/qb_$c.log 2>&1
  tail -1 gpurun_out/qb_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg%s'%$c, 'x$REP', 'ms', round(d['ms_per_step'],4), 'Gsteps/s', round(d['value']/1e9,2), d['roofline']['bound'], 'frac', round(d['roofline']['frac'],4))" || tail -4 gpurun_out/qb_$c.log
done
