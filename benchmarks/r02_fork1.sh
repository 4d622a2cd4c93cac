cd $GRAFT_REPO_ROOT
for c in c2 c3; do for r in 1 2 3 4 5; do for f in 0 1; do
  MOE_BWD_FORK=$f timeout 300 python bench.py --config $c --no-cpu --no-ring --no-e2e --steps 20 > gpurun_out/fork1_${c}_${f}_${r}.json 2>/dev/null
  python - gpurun_out/fork1_${c}_${f}_${r}.json $f $c <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[3], "fork", sys.argv[2], "%.3f ms" % d["ms_per_step"], d["clocks"]["sm_mhz"])
PY
done; done; done
