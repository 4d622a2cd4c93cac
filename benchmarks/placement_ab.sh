timeout 900 python -m pytest tests/test_ep_gpu.py tests/test_layer_gpu.py -x -q > gpurun_out/r01p_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r01p_pytest.log
for n in 2 4; do for pl in contiguous round_robin; do for c in c3 c2; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700+n)) bench.py --gpus $n --config $c --no-cpu --placement $pl > gpurun_out/r01p_${c}_n${n}_${pl}.json 2> gpurun_out/r01p_${c}_n${n}_${pl}.err; echo "$c n$n $pl rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r01p_${c}_n${n}_${pl}.json').read().strip().splitlines()[-1]); print('   %.2fM %.3fms frac=%.3f'%(d['value']/1e6, d['ms_per_step'], d['roofline']['frac']))"
done; done; done
