cd $GRAFT_REPO_ROOT
S="ffn1 shape  K-major  bf16 STORE,ffn2,GELU,wgrad"
echo "== shared-b"; python benchmarks/gemm_sweep.py --only "ffn1 shape  K-major  bf16 STORE,ffn2" --groups 64 --rows 1024 --shared-b
for r in 1 2; do for v in base pf8 pf16 pf32; do
  echo "== $v 64x1024 ($r)"; MOE_B200_LIB=exp/$v/libmoe_b200.so python benchmarks/gemm_sweep.py --only "$S" --groups 64 --rows 1024
done; done
for v in base pf16; do echo "== $v 64x1030"; MOE_B200_LIB=exp/$v/libmoe_b200.so python benchmarks/gemm_sweep.py --only "ffn1 shape  K-major  bf16 STORE,ffn2" --groups 64 --rows 1030; done
bash benchmarks/ab_bench.sh c2 2 base pf8 pf16 pf32
