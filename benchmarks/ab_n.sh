# A/B two builds at N = all GPUs of the box: benchmarks/ab_n.sh LIB_A LIB_B [rounds]
A=$1; B=$2; R=${3:-2}; NG=$(nvidia-smi -L | wc -l)
for r in $(seq 1 $R); do for L in "$A" "$B"; do
MOE_B200_LIB=$L timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29850 bench.py --gpus $NG --config ${CONFIG:-c2} --no-cpu --no-e2e --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms_per_step']
print('$L'[-30:].ljust(30), '%.2fM'%(d['value']/1e6), '%.3fms'%d['ms_per_step'], ' '.join('%s=%.3f'%(k.split('.')[1][:12],p[k]) for k in ('bwd.allreduce_gate','bwd.gate_wgrad','fwd.dispatch_p2p','bwd.combine_bwd','fwd.a2a_combine')))"
done; done
