cd $GRAFT_REPO_ROOT
for c in c2 c3; do for r in 1 2 3; do for v in hn2 hn1 hd1; do
  MOE_B200_LIB=exp/$v/libmoe_b200.so timeout 300 python bench.py --config $c --no-cpu --no-ring --no-e2e --steps 10 > gpurun_out/hn_${c}_${v}_${r}.json 2>/dev/null
  python - gpurun_out/hn_${c}_${v}_${r}.json $v $c <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[3], sys.argv[2], "%.3f ms" % d["ms_per_step"], [(g["gemm"], round(g["ms"]*1e3)) for g in d["roofline"]["per_gemm"]], d["clocks"]["sm_mhz"])
PY
done; done; done
