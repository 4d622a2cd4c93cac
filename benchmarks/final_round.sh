# End-of-round sweep on one box (N GPUs): GPU tests, every config at N=1 and
# N=2..NG, the reference arm, and the ncu evidence on GPU 0.
TAG=${1:-r01z}; PROFILE=${2:-1}
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv,noheader | head -1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/${TAG}_pytest_gpu.log
timeout 400 python bench.py --timeline gpurun_out/${TAG}_c2_n1_timeline.json > gpurun_out/${TAG}_c2_n1.json 2> gpurun_out/${TAG}_c2_n1.err; echo "c2 n1 rc=$?"
timeout 400 python bench.py --impl reference > gpurun_out/${TAG}_reference_n1.json 2> gpurun_out/${TAG}_reference_n1.err; echo "ref rc=$?"
for c in c1 c3 c4; do
  timeout 300 python bench.py --config $c --no-cpu > gpurun_out/${TAG}_${c}_n1.json 2> gpurun_out/${TAG}_${c}_n1.err; echo "$c n1 rc=$?"
done
n=2
while [ $n -le $NG ]; do
  for c in c2 c1 c3 c4; do
    X=$( [ $c = c2 ] || echo --no-cpu )
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29600 + n)) bench.py --gpus $n --config $c $X > gpurun_out/${TAG}_${c}_n$n.json \
      2> gpurun_out/${TAG}_${c}_n$n.err; echo "$c n$n rc=$?"
  done
  n=$((n * 2))
done
if [ "$PROFILE" = 1 ]; then CUDA_VISIBLE_DEVICES=0 bash benchmarks/profile_round.sh ${TAG} c2; fi
