mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_ep_gpu.py -x -q > gpurun_out/r02n_ep.log 2>&1; echo "ep rc=$?"; tail -2 gpurun_out/r02n_ep.log
timeout 300 python -m pytest tests/test_layer_gpu.py tests/test_moe_golden_gpu.py -x -q -k "f32 or fp32 or c1" > gpurun_out/r02n_l.log 2>&1; echo "layer rc=$?"; tail -1 gpurun_out/r02n_l.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29537 bench.py --gpus 2 --config c1 --no-cpu > gpurun_out/r02n_c1_n2.json 2> gpurun_out/r02n_c1_n2.err; echo "c1 n2 rc=$?"
