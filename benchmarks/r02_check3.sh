mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_ep_gpu.py -x -q -k "stack" > gpurun_out/r02h_ep.log 2>&1; echo "ep rc=$?"; tail -2 gpurun_out/r02h_ep.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c4 --no-cpu > gpurun_out/r02h_c4_n2.json 2> gpurun_out/r02h_c4_n2.err; echo "c4 n2 rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 300 ncu --set full --clock-control none -k "regex:seg_colsum|sum_parts" -s 2 -c 2 -o gpurun_out/r02h_red python bench.py --config c2 --steps 1 --warmup 3 --no-cpu --no-e2e --no-ring > gpurun_out/r02h_ncu.log 2>&1; echo "ncu rc=$?"
