#!/bin/bash
# exit-ring A/B (cfg1): tests touching the source-free kernels per library, library A/B, refill sweep
#   LIBS="lib1 lib2 ..." [SWEEP="5 7 9"] [SWEEPLIB=lib] bash profiles/ab_exit_ring.sh
for lib in $(echo $LIBS | tr ' ' '\n' | sort -u); do
  echo "== tests with $lib"
  WOS_B200_LIB=$PWD/paper_2603_01193_b200/$lib python -m pytest tests -m gpu -x -q -k "sourcefree or fuzz or native or shard" 2>&1 | tail -2
done
bash profiles/ab_libs.sh "1" $LIBS
for r in ${SWEEP:-}; do
  WOS_B200_LIB=$PWD/paper_2603_01193_b200/${SWEEPLIB:-libwos_b200.so} timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config 1 --replicas 16 --refill-min $r > gpurun_out/rf.log 2>&1
  tail -1 gpurun_out/rf.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('refill_min $r', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4))" || tail -3 gpurun_out/rf.log
done
