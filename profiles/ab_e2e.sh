#!/bin/bash
# cfg4 device and e2e rates of library variants: ab_e2e.sh lib1 lib2 ...
for lib in "$@"; do
  WOS_B200_LIB=$PWD/paper_2603_01193_b200/$lib timeout 180 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/abe.log 2>&1
  tail -1 gpurun_out/abe.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'ms', round(d['ms_per_step'],4), 'value %.4g e2e %.4g ratio %.4f' % (d['value'], d['e2e']['value'], d['e2e']['value']/d['value']))" || tail -3 gpurun_out/abe.log
done
