cd $GRAFT_REPO_ROOT
MOE_B200_LIB=exp/g1/libmoe_b200.so timeout 900 python -m pytest tests/test_layer_gpu.py tests/test_moe_golden_gpu.py -x -q 2>&1 | tail -2
for r in 1 2 3; do for v in g0 g1; do
  MOE_B200_LIB=exp/$v/libmoe_b200.so timeout 300 python bench.py --config c1 --no-cpu --no-ring --no-e2e --steps 20 > gpurun_out/gf_${v}_${r}.json 2>/dev/null
  python - gpurun_out/gf_${v}_${r}.json $v <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
h = {k["kernel"]: round(k["us"], 1) for k in d["roofline"]["hbm_kernels"]}
print("c1", sys.argv[2], "%.3f ms" % d["ms_per_step"], h.get("gate_wgrad"), h.get("gate_dgrad_gather_dx"), d["clocks"]["sm_mhz"])
PY
done; done
