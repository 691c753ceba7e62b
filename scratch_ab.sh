# A/B of library variants: scratch_ab.sh "name=lib ..." "bench args" 
set -u
LIBS="$1"; ARGS="$2"; REP=${3:-1}
for r in $(seq 1 $REP); do
for kv in $LIBS; do
  n=${kv%%=*}; lib=${kv#*=}
  for c in $ARGS; do
    cc=${c%%:*}; rr=${c#*:}
    WOS_B200_LIB=$lib timeout 120 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras --config $cc --replicas $rr > gpurun_out/ab_${n}_$cc.log 2>&1
    tail -1 gpurun_out/ab_${n}_$cc.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n cfg$cc', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4))" || tail -3 gpurun_out/ab_${n}_$cc.log
  done
done
done
