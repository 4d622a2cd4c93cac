mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_ep_gpu.py -x -q -k "stack or matches_single" > gpurun_out/r02g_ep.log 2>&1; echo "ep rc=$?"; tail -2 gpurun_out/r02g_ep.log
timeout 300 python -m pytest tests/test_layer_gpu.py -x -q -k "stack or deterministic or host" > gpurun_out/r02g_layer.log 2>&1; echo "layer rc=$?"; tail -2 gpurun_out/r02g_layer.log
timeout 300 python bench.py --config c2 --no-cpu --no-ring > gpurun_out/r02g_c2_n1.json 2> gpurun_out/r02g_c2_n1.err; echo "c2 rc=$?"
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c4 --no-cpu > gpurun_out/r02g_c4_n2.json 2> gpurun_out/r02g_c4_n2.err; echo "c4 n2 rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02g_launches.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e --no-ring > /dev/null 2>&1; echo "ncu rc=$?"
