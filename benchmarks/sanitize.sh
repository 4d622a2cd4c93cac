# compute-sanitizer over the small GPU tests (memcheck, racecheck, synccheck,
# initcheck): routing, grouped GEMM (tcgen05 + SIMT), the layer fwd+bwd and
# the data-plane ops.  Logs -> gpurun_out/${TAG}_sanitize_<tool>.log
TAG=${1:-r02}
mkdir -p gpurun_out
SEL="tests/test_routing_gpu.py::test_routing_ties_nan_inf tests/test_routing_gpu.py::test_routing_zero_capacity \
tests/test_routing_gpu.py::test_routing_bit_exact \
tests/test_gemm_gpu.py tests/test_moesim_gpu.py \
tests/test_layer_gpu.py::test_layer_bf16_top2_small tests/test_layer_gpu.py::test_layer_fp32_drops \
tests/test_layer_gpu.py::test_layer_ragged_tokens_bf16 tests/test_layer_gpu.py::test_layer_bf16_skewed_drops_c3"
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check full"
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 50 \
    --error-exitcode 99 python -m pytest $SEL -q -x -p no:cacheprovider \
    > gpurun_out/${TAG}_sanitize_${tool}.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/${TAG}_sanitize_${tool}.log | tail -3 | tr '\n' ' ')"
done
