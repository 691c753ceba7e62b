for lib in libwos_b200.so libwos_ds1.so libwos_ds2.so; do
WOS_B200_LIB=$PWD/paper_2603_01193_b200/$lib timeout 120 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-extras --config 3 > gpurun_out/ds.log 2>&1
tail -1 gpurun_out/ds.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); w=d['roofline']['work']; print('$lib', d['ms_per_step'], w.get('segments_per_step'), w.get('seg_evals'))" || tail -3 gpurun_out/ds.log
done
