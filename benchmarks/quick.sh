# quick GPU check: GEMM + layer GPU tests, then c2 (and optional configs) at N=1
TAG=${1:-q}; shift; CFGS=${@:-c2}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_layer_gpu.py tests/test_moe_golden_gpu.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
for c in $CFGS; do
  timeout 300 python bench.py --config $c --no-cpu --no-ring > gpurun_out/${TAG}_${c}.json 2> gpurun_out/${TAG}_${c}.err; echo "$c rc=$?"
  python - gpurun_out/${TAG}_${c}.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d["roofline"]
print("%.3fM tok/s %.3f ms/step frac=%.3f e2e=%.3fM" % (d["value"]/1e6, d["ms_per_step"], r["frac"], d["e2e"]["value"]/1e6), d["clocks"])
print("  ", {g["gemm"]: round(g["ms"], 3) for g in r["per_gemm"]})
print("  ", {k["kernel"]: round(k["us"], 1) for k in r["hbm_kernels"]})
PY
done
