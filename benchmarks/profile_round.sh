# ncu evidence for one round (1 GPU, config c2 unless given):
#   launch list of the bench step, --set full of the nine tc_gemm launches and
#   the eight small kernels of one step.  Read back with profiles/ncu_summary.py.
TAG=${1:-r01}; C=${2:-c2}
mkdir -p gpurun_out
B="python bench.py --config $C --steps 1 --warmup 3 --no-cpu --no-e2e --no-ring"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --config $C --steps 2 --warmup 3 --no-cpu --no-e2e --no-ring \
  > gpurun_out/${TAG}_launches.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -s 27 -c 9 \
  -o gpurun_out/prof_${TAG} $B > gpurun_out/${TAG}_prof.log 2>&1; echo "gemm capture rc=$?"
timeout 900 ncu --set full --clock-control none -k "regex:route|dispatch|combine|colsum" -s 24 -c 8 \
  -o gpurun_out/prof_${TAG}_small $B > gpurun_out/${TAG}_prof_small.log 2>&1; echo "small capture rc=$?"
