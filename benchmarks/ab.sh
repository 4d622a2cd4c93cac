#!/bin/bash
# A/B two builds of libmoe_b200.so on the same GPU: alternates runs of
# bench.py and prints value + selected phases.  Usage: benchmarks/ab.sh LIB_A LIB_B [rounds]
A=$1; B=$2; R=${3:-2}
for r in $(seq 1 $R); do
  for L in "$A" "$B"; do
    MOE_B200_LIB=$L python bench.py --config ${CONFIG:-c2} --steps ${STEPS:-20} --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms_per_step']
keys=['fwd.route','bwd.route_bwd','fwd.ffn1','fwd.ffn2','bwd.dgrad_ffn2','bwd.dgrad_ffn1','bwd.wgrad_w1','bwd.wgrad_w2','fwd.dispatch','fwd.combine','bwd.combine_bwd','bwd.gate_dgrad_gather_dx','bwd.bias_grads']
print('$(basename $L)'[:16].ljust(16), '%.2fM'%(d['value']/1e6), '%.3fms'%d['ms_per_step'], 'sum=%.3f'%sum(p.values()), 'mhz=%s'%d['clocks'].get('sm_mhz'), ' '.join('%s=%.3f'%(k.split('.')[1][:10],p.get(k,0)) for k in keys))"
  done
done
