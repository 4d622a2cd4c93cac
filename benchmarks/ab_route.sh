timeout 300 python -m pytest tests/test_routing_gpu.py tests/test_moe_golden_gpu.py tests/test_layer_gpu.py -q -x 2>&1 | tail -1
for r in 1 2; do for v in r256 r128; do
  MOE_B200_LIB=exp/$v/libmoe_b200.so timeout 300 python bench.py --config c2 --no-cpu --no-ring --no-e2e --steps 10 > gpurun_out/abr_${v}_${r}.json 2>/dev/null
  python - gpurun_out/abr_${v}_${r}.json $v <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
ph = {k["kernel"]: round(k["us"], 1) for k in d["roofline"]["hbm_kernels"]}
print(sys.argv[2], "%.3f ms" % d["ms_per_step"], ph.get("route"), ph.get("route_bwd"), d["clocks"]["sm_mhz"])
PY
done; done
