#!/bin/bash
# Refresh every measurement under profiles/ (run under gpurun, one GPU). $1 = tag
# The ncu reports are summarised on the box (summarize_ncu.py, sass_hot.py) and only the
# cfg4 report is kept: gpurun brings back at most 64 MiB.
set -u
TAG=${1:-r2}
python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err; tail -1 gpurun_out/bench_full.log > gpurun_out/${TAG}_bench_cfg4.json
python bench.py --impl reference > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref.log > gpurun_out/${TAG}_bench_reference_arm.json
bash profiles/quick_bench.sh "4 3 0 1 2" > gpurun_out/${TAG}_configs.txt 2>&1
bash profiles/ncu_cmds.sh $TAG
python profiles/summarize_ncu.py gpurun_out/prof_${TAG}.ncu-rep > gpurun_out/${TAG}_cfg4_ncu_full.txt 2>&1
S=$(python -c "import json; print(int(json.load(open('gpurun_out/${TAG}_bench_cfg4.json'))['walk_steps_per_step']))")
ncu -i gpurun_out/prof_${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_${TAG}.csv 2>/dev/null
python profiles/sass_hot.py gpurun_out/sass_${TAG}.csv $S > gpurun_out/${TAG}_cfg4_sass.txt; rm -f gpurun_out/sass_${TAG}.csv
cp gpurun_out/launches_${TAG}.csv gpurun_out/${TAG}_cfg4_launches.csv
for c in "3 1" "1 16" "2 16" "0 64"; do
  set -- $c
  bash profiles/ncu_cfg.sh $TAG $1 $2
  python profiles/summarize_ncu.py gpurun_out/prof_${TAG}_c$1.ncu-rep > gpurun_out/${TAG}_cfg$1_ncu_full.txt 2>&1
  rm -f gpurun_out/prof_${TAG}_c$1.ncu-rep
done
for b in screened polar mesh; do timeout 600 python profiles/bench_$b.py > gpurun_out/${TAG}_$b.txt 2>&1; done
ls -la gpurun_out/
