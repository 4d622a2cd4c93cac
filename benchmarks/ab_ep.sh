# interleaved multi-GPU bench A/B of variant libraries: bash benchmarks/ab_ep.sh CONFIG ROUNDS v1 v2 ...
C=$1; R=$2; shift 2
NG=$(nvidia-smi -L | wc -l)
for r in $(seq 1 $R); do for v in "$@"; do
  MOE_B200_LIB=exp/$v/libmoe_b200.so timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus $NG --config $C --no-cpu --no-e2e > gpurun_out/abe_${v}_${r}.json 2>/dev/null
  python - gpurun_out/abe_${v}_${r}.json $v <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
ph = d["phases_ms_per_step"]
print(sys.argv[2], "%.2fM" % (d["value"] / 1e6), "%.3f ms" % d["ms_per_step"], {k: round(v, 3) for k, v in ph.items() if "a2a" in k or "dispatch" in k or "combine_bwd" in k}, round(d["nvlink"]["achieved"]))
PY
done; done
