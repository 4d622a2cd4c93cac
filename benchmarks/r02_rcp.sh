cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in rcp0 rcp1; do echo "== $v ($r)"; MOE_B200_LIB=exp/$v/libmoe_b200.so timeout 120 python benchmarks/gemm_sweep.py --only "GELU" --groups 64 --rows 1024; done; done
MOE_B200_LIB=exp/rcp1/libmoe_b200.so timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_layer_gpu.py tests/test_moe_golden_gpu.py -x -q 2>&1 | tail -2
for r in 1 2 3 4 5; do for v in rcp0 rcp1; do
  MOE_B200_LIB=exp/$v/libmoe_b200.so timeout 300 python bench.py --config c2 --no-cpu --no-ring --no-e2e --steps 20 > gpurun_out/rcp_${v}_${r}.json 2>/dev/null
  python - gpurun_out/rcp_${v}_${r}.json $v <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("c2", sys.argv[2], "%.3f ms" % d["ms_per_step"], [(g["gemm"], round(g["ms"]*1e3)) for g in d["roofline"]["per_gemm"]][:1], d["clocks"]["sm_mhz"])
PY
done; done
