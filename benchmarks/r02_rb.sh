cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for c in c2 c3 c1; do for r in 1 2; do for v in rbold rbwarp; do
  MOE_B200_LIB=exp/$v/libmoe_b200.so timeout 300 python bench.py --config $c --no-cpu --no-ring --no-e2e --steps 10 > gpurun_out/rb_${c}_${v}_${r}.json 2>/dev/null
  python - gpurun_out/rb_${c}_${v}_${r}.json $v $c <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
h = {k["kernel"]: (round(k["us"], 1), round(k["frac"], 2)) for k in d["roofline"]["hbm_kernels"]}
print(sys.argv[3], sys.argv[2], "%.3f ms" % d["ms_per_step"], h["route_bwd"], d["clocks"]["sm_mhz"])
PY
done; done; done
