cd $GRAFT_REPO_ROOT
MOE_B200_LIB=exp/sc1/libmoe_b200.so timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in c2 c3; do for r in 1 2 3; do for v in sc0 sc1; do
  MOE_B200_LIB=exp/$v/libmoe_b200.so timeout 300 python bench.py --config $c --no-cpu --no-ring --no-e2e --steps 20 > gpurun_out/sc_${c}_${v}_${r}.json 2>/dev/null
  python - gpurun_out/sc_${c}_${v}_${r}.json $v $c <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
ph = d["phases_ms_per_step"]
print(sys.argv[3], sys.argv[2], "%.3f ms" % d["ms_per_step"], "dgrad2 phase %.1f" % (ph["bwd.dgrad_ffn2"]*1e3), d["clocks"]["sm_mhz"])
PY
done; done; done
