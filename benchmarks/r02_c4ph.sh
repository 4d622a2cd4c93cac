cd $GRAFT_REPO_ROOT
for pdl in 1 0; do
MOE_PDL=$pdl timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu --no-ring --no-e2e > gpurun_out/c4ph_$pdl.json 2>gpurun_out/c4ph_$pdl.err
python - gpurun_out/c4ph_$pdl.json $pdl <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("PDL", sys.argv[2], d["ms_per_step"], d["clocks"])
print({k: round(v*1e3,1) for k, v in d["phases_ms_per_step"].items()})
PY
done
