# interleaved bench A/B of variant libraries on one config: bash benchmarks/ab_bench.sh CONFIG ROUNDS v1 v2 ...
C=$1; R=$2; shift 2
for r in $(seq 1 $R); do for v in "$@"; do
  MOE_B200_LIB=exp/$v/libmoe_b200.so timeout 300 python bench.py --config $C --no-cpu --no-ring --no-e2e --steps 10 > gpurun_out/ab_${v}_${r}.json 2>/dev/null
  python - gpurun_out/ab_${v}_${r}.json $v <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
ph = {k["kernel"]: round(k["us"], 1) for k in d["roofline"]["hbm_kernels"]}
print(sys.argv[2], "%.3f ms" % d["ms_per_step"], ph.get("gate_dgrad_gather_dx"), d["clocks"]["sm_mhz"])
PY
done; done
