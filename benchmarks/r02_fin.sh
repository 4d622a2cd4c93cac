cd $GRAFT_REPO_ROOT
MOE_B200_LIB=exp/fcs2/libmoe_b200.so timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for r in 1 2 3; do for v in fold fcs2; do
  MOE_B200_LIB=exp/$v/libmoe_b200.so timeout 300 python bench.py --config c1 --no-cpu --no-ring --no-e2e --steps 20 > gpurun_out/fin_${v}_${r}.json 2>/dev/null
  python - gpurun_out/fin_${v}_${r}.json $v <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], "%.3f ms" % d["ms_per_step"], "%.3fM" % (d["value"]/1e6), [(g["gemm"], round(g["ms"]*1e3)) for g in d["roofline"]["per_gemm"]], d["clocks"]["sm_mhz"])
PY
done; done
