# A/B one build under two environment settings: benchmarks/ab_env.sh "VAR=a" "VAR=b" [rounds]
A=$1; B=$2; R=${3:-2}
for r in $(seq 1 $R); do
  for V in "$A" "$B"; do
    env $V python bench.py --config ${CONFIG:-c2} --steps ${STEPS:-20} --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms_per_step']
print('$V'.ljust(18), '%.3fM'%(d['value']/1e6), '%.3fms'%d['ms_per_step'], ' '.join('%s=%.3f'%(k.split('.')[1][:10],v) for k,v in sorted(p.items()) if v > 0.02))"
  done
done
