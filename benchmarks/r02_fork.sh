cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in c2 c3 c1; do for r in 1 2 3; do for f in 0 1; do
  MOE_BWD_FORK=$f timeout 300 python bench.py --config $c --no-cpu --no-ring --no-e2e --steps 20 > gpurun_out/fork_${c}_${f}_${r}.json 2>/dev/null
  python - gpurun_out/fork_${c}_${f}_${r}.json $f $c <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[3], "fork", sys.argv[2], "%.3f ms" % d["ms_per_step"], d["clocks"]["sm_mhz"])
PY
done; done; done
for f in 0 1; do MOE_BWD_FORK=$f timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --config c2 --no-cpu --no-ring --no-e2e --steps 20 > gpurun_out/fork_n2_${f}.json 2>/dev/null; python - gpurun_out/fork_n2_${f}.json $f <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("c2 N=2 fork", sys.argv[2], "%.3f ms" % d["ms_per_step"], "%.2fM" % (d["value"]/1e6))
PY
done
