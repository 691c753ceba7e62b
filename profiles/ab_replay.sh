#!/bin/bash
# REPLAY_F64 throughput of library variants (cfg4 and cfg1 in replay mode): ab_replay.sh lib1 lib2 ...
for lib in "$@"; do
  for c in 4 1 3; do
    WOS_B200_LIB=$PWD/paper_2603_01193_b200/$lib timeout 300 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-extras --config $c --mode replay 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib cfg$c replay ms', round(d['ms_per_step'],3), 'walk-steps/s %.4g' % d['value'])"
  done
done
