cd $GRAFT_REPO_ROOT
S="ffn1 shape  K-major  bf16 STORE,ffn2,GELU,dgrad2 shp  B MN     bf16 DGELU,dgrad1,wgrad"
echo "== sweep mc (first run, 60s cap)"; timeout 60 python benchmarks/gemm_sweep.py --only "ffn2" --groups 64 --rows 1024 --reps 3; echo rc=$?
timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -5
for r in 1 2; do for m in 0 1; do
  echo "== MC=$m 64x1024 ($r)"; MOE_GEMM_MC=$m timeout 120 python benchmarks/gemm_sweep.py --only "$S" --groups 64 --rows 1024
done; done
for m in 0 1; do echo "== MC=$m 64x1030"; MOE_GEMM_MC=$m timeout 120 python benchmarks/gemm_sweep.py --only "ffn1 shape  K-major  bf16 STORE,ffn2" --groups 64 --rows 1030; done
echo "== MC=1 dense"; timeout 120 python benchmarks/gemm_sweep.py --only "ffn1 shape  K-major  bf16 STORE,ffn2" --groups 1 --rows 65536
timeout 900 python -m pytest tests/test_layer_gpu.py -x -q 2>&1 | tail -5
for r in 1 2; do for m in 0 1; do
  MOE_GEMM_MC=$m timeout 300 python bench.py --config c2 --no-cpu --no-ring --no-e2e --steps 10 > gpurun_out/mc_${m}_${r}.json 2>/dev/null
  python - gpurun_out/mc_${m}_${r}.json $m <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("MC", sys.argv[2], "%.3f ms" % d["ms_per_step"], [(g["gemm"], round(g["ms"]*1e3)) for g in d["roofline"]["per_gemm"]], d["clocks"]["sm_mhz"])
PY
done; done
