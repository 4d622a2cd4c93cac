mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x -k split > gpurun_out/r02i_gemm.log 2>&1; echo "gemm rc=$?"; tail -3 gpurun_out/r02i_gemm.log
timeout 600 python -m pytest tests/test_layer_gpu.py tests/test_moe_golden_gpu.py -q -x -k "fp32 or f32 or layer_c1 or golden or deterministic" > gpurun_out/r02i_layer.log 2>&1; echo "layer rc=$?"; tail -3 gpurun_out/r02i_layer.log
timeout 300 python bench.py --config c1 --no-cpu --no-ring > gpurun_out/r02i_c1.json 2> gpurun_out/r02i_c1.err; echo "c1 rc=$?"
