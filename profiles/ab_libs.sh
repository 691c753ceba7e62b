#!/bin/bash
# A/B libs: ab.sh "cfgs" lib1 lib2 ...
CFGS=$1; shift
for lib in "$@"; do
  for c in $CFGS; do
    case $c in 0) REP=64;; 1) REP=16;; 2) REP=16;; *) REP=1;; esac
    WOS_B200_LIB=$PWD/paper_2603_01193_b200/$lib timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $c --replicas $REP > gpurun_out/ab.log 2>&1
    tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'cfg$c', 'ms', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4))" || tail -3 gpurun_out/ab.log
  done
done
