#!/bin/bash
# ncu --set full capture of one walk launch of a BASELINE config (run under gpurun, one GPU)
#   bash profiles/ncu_cfg.sh <tag> <config> [replicas]
set -u
TAG=$1; C=$2; R=${3:-1}
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extras --config $C --replicas $R"
$CMD > gpurun_out/plain_${TAG}_c$C.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:wos_walk_kernel -s 1 -c 1 \
    -o gpurun_out/prof_${TAG}_c$C $CMD > gpurun_out/ncu_${TAG}_c$C.log 2>&1
echo "cfg$C ncu rc=$?"
