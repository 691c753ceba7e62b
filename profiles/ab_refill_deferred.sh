#!/bin/bash
# per-config time against the deferred-recording refill threshold (runtime tuning, no rebuild)
#   bash profiles/ab_refill_deferred.sh "<configs>" d1 d2 ...
CFGS=$1; shift
for c in $CFGS; do
  case $c in 0) REP=64;; 1) REP=16;; 2) REP=16;; *) REP=1;; esac
  for r in "$@"; do
    timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras --config $c --replicas $REP --refill-min-deferred $r > gpurun_out/rfd.log 2>&1
    tail -1 gpurun_out/rfd.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg$c refill_min_deferred $r', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4))" || tail -3 gpurun_out/rfd.log
  done
done
