#!/bin/bash
# Refresh every measurement under profiles/ (run under gpurun, one GPU). $1 = tag
set -u
TAG=${1:-r1d}
python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err; tail -1 gpurun_out/bench_full.log > gpurun_out/${TAG}_bench_cfg4.json
python bench.py --impl reference > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref.log > gpurun_out/${TAG}_bench_reference_arm.json
bash profiles/quick_bench.sh "4 3 0 1 2" > gpurun_out/${TAG}_configs.txt 2>&1
bash profiles/ncu_cmds.sh $TAG
bash profiles/ncu_cfg3.sh
for b in screened polar mesh; do timeout 600 python profiles/bench_$b.py > gpurun_out/${TAG}_$b.txt 2>&1; done
ls -la gpurun_out/
