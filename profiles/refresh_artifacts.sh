set -u
python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err; tail -1 gpurun_out/bench_full.log > gpurun_out/bench_full.json
python bench.py --impl reference > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref.log > gpurun_out/bench_ref.json
bash profiles/ncu_cmds.sh r1h
bash profiles/ncu_cfg3.sh
ls -la gpurun_out/
