# One GPU session of the round: GPU tests, bench lines, optional ncu captures.
# usage: bash benchmarks/gpu_round.sh TAG [tests|notests] [configs...]
TAG=${1:-x}; TESTS=${2:-tests}; shift 2; CFGS=${@:-c2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv,noheader
NG=$(nvidia-smi -L | wc -l)
if [ "$TESTS" = tests ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -3 gpurun_out/${TAG}_pytest_gpu.log
fi
for c in $CFGS; do
  timeout 300 python bench.py --config $c $( [ $c = c2 ] || echo --no-cpu ) > gpurun_out/${TAG}_${c}_n1.json 2> gpurun_out/${TAG}_${c}_n1.err; echo "$c n1 rc=$?"
  if [ $NG -ge 2 ]; then
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $NG --config $c --no-cpu > gpurun_out/${TAG}_${c}_n$NG.json 2> gpurun_out/${TAG}_${c}_n$NG.err; echo "$c n$NG rc=$?"
  fi
done
for f in gpurun_out/${TAG}_*.json; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
except Exception as e:
    print(f, "unreadable", e); sys.exit()
r = d.get("roofline", {})
print(f, "%.3fM" % (d["value"] / 1e6), "%.3fms" % d["ms_per_step"], "frac=%.3f" % r.get("frac", 0),
      "e2e=%s" % (d.get("e2e") or {}).get("value"), d.get("clocks"))
print("   ", {k: round(v, 3) for k, v in d.get("phases_ms_per_step", {}).items()})
PY
done
