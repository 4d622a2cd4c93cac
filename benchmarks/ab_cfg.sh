# interleaved bench A/B of variant libraries: bash benchmarks/ab_cfg.sh CONFIG ROUNDS v1 v2 ...
C=$1; R=$2; shift 2
for r in $(seq 1 $R); do for v in "$@"; do
  MOE_B200_LIB=exp/$v/libmoe_b200.so timeout 300 python bench.py --config $C --no-cpu --no-ring --no-e2e --steps 10 > gpurun_out/abc_${v}_${r}.json 2>/dev/null
  python - gpurun_out/abc_${v}_${r}.json $v <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
g = {x["gemm"]: round(x["ms"], 3) for x in d["roofline"]["per_gemm"]}
print(sys.argv[2], "%.2fM" % (d["value"] / 1e6), "%.3f ms" % d["ms_per_step"], g.get("wgrad_w1"), g.get("wgrad_w2"), d["clocks"]["sm_mhz"])
PY
done; done
