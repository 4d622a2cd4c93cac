cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in sgen sarith; do echo "== $v ($r)"; MOE_B200_LIB=exp/$v/libmoe_b200.so timeout 120 python benchmarks/gemm_sweep.py --only "ffn1 shape  K-major  bf16 STORE,GELU,ffn2,DGELU,wgrad" --groups 64 --rows 1024; MOE_B200_LIB=exp/$v/libmoe_b200.so timeout 120 python benchmarks/gather_bench.py --only c2,c3,c4; done; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in c2 c3 c1; do for r in 1 2; do for v in sgen sarith; do
  MOE_B200_LIB=exp/$v/libmoe_b200.so timeout 300 python bench.py --config $c --no-cpu --no-ring --no-e2e --steps 10 > gpurun_out/sa_${c}_${v}_${r}.json 2>/dev/null
  python - gpurun_out/sa_${c}_${v}_${r}.json $v $c <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[3], sys.argv[2], "%.3f ms" % d["ms_per_step"], [(g["gemm"], round(g["ms"]*1e3)) for g in d["roofline"]["per_gemm"]], {k["kernel"]: round(k["us"], 1) for k in d["roofline"]["hbm_kernels"]}.get("gate_dgrad_gather_dx"), d["clocks"]["sm_mhz"])
PY
done; done; done
