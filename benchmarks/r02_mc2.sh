cd $GRAFT_REPO_ROOT
for c in c2 c1 c3; do for r in 1 2; do for m in 0 1; do
  MOE_GEMM_MC=$m timeout 300 python bench.py --config $c --no-cpu --no-ring --no-e2e --steps 10 > gpurun_out/mc_${c}_${m}_${r}.json 2>/dev/null
  python - gpurun_out/mc_${c}_${m}_${r}.json $m $c <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[3], "MC", sys.argv[2], "%.3f ms" % d["ms_per_step"], [(g["gemm"], round(g["ms"]*1e3)) for g in d["roofline"].get("per_gemm", [])], d["clocks"]["sm_mhz"])
PY
done; done; done
