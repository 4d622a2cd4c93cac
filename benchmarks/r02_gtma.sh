cd $GRAFT_REPO_ROOT
echo "== first run (60s cap)"; timeout 60 python benchmarks/gather_bench.py --only c2 --reps 3; echo rc=$?
for r in 1 2; do for v in gcp gtma2; do echo "== $v ($r)"; MOE_B200_LIB=exp/$v/libmoe_b200.so timeout 120 python benchmarks/gather_bench.py --only c2,c3,c4; done; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for r in 1 2; do for v in gcp gtma2; do
  MOE_B200_LIB=exp/$v/libmoe_b200.so timeout 300 python bench.py --config c2 --no-cpu --no-ring --no-e2e --steps 10 > gpurun_out/gt_${v}_${r}.json 2>/dev/null
  python - gpurun_out/gt_${v}_${r}.json $v <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], "%.3f ms" % d["ms_per_step"], {k["kernel"]: round(k["us"], 1) for k in d["roofline"]["hbm_kernels"]}["gate_dgrad_gather_dx"], d["clocks"]["sm_mhz"])
PY
done; done
