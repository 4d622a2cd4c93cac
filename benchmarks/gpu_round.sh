set -x
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r01g_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r01g_pytest_gpu.log
python bench.py > gpurun_out/r01g_c2_n1.json 2> gpurun_out/r01g_c2_n1.err; echo rc=$?
for c in c1 c3 c4; do timeout 300 python bench.py --config $c --no-cpu > gpurun_out/r01g_${c}_n1.json 2> gpurun_out/r01g_${c}_n1.err; echo $c rc=$?; done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/r01g_c2_n2.json 2> gpurun_out/r01g_c2_n2.err; echo n2 rc=$?
for c in c3 c4; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --config $c --no-cpu --no-e2e > gpurun_out/r01g_${c}_n2.json 2> gpurun_out/r01g_${c}_n2.err; echo $c n2 rc=$?; done
cat gpurun_out/r01g_*.json | cut -c1-400
