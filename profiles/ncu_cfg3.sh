CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --config 3"
$CMD > gpurun_out/plain_c3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:wos_walk_kernel -s 1 -c 1 -o gpurun_out/prof_c3 $CMD > gpurun_out/ncu_c3.log 2>&1; echo ncu=$?
