# A/B the GEMM micro-benchmark over variant libraries: bash benchmarks/ab_sweep.sh v1 v2 ...
for v in "$@"; do
  echo "== $v"
  MOE_B200_LIB=exp/$v/libmoe_b200.so timeout 300 python benchmarks/gemm_sweep.py --reps 30
done
