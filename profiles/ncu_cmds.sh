#!/bin/bash
# ncu recipes used for profiles/ (run under gpurun, one GPU). $1 = tag
set -u
TAG=${1:-r1}
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:wos_walk_kernel -s 1 -c 1 -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu rc=$?"
