# ncu --set full capture of one kernel of the c2 step (1 GPU), e.g.
#   bash benchmarks/ncu_kernel.sh TAG 'regex:256, 0, 1, 0, 4' [config]
TAG=$1; K=$2; C=${3:-c2}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "$K" -s 2 -c 1 -o gpurun_out/${TAG} python bench.py --config $C --steps 1 --warmup 1 --no-cpu --no-e2e --no-ring \
  > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/${TAG}_ncu.log
