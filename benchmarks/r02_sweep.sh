set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
python benchmarks/gemm_sweep.py --only "ffn1 shape  K-major  bf16 STORE,ffn2,GELU" --groups 64 --rows 1024 --cublas
python benchmarks/gemm_sweep.py --only "ffn1 shape  K-major  bf16 STORE,ffn2,GELU" --groups 1 --rows 65536
python benchmarks/gemm_sweep.py --only "ffn1 shape  K-major  bf16 STORE,ffn2" --groups 8 --rows 8192
python benchmarks/gemm_sweep.py --only "ffn1 shape  K-major  bf16 STORE,ffn2" --groups 64 --rows 1030
python benchmarks/gemm_sweep.py --only "ffn1 shape  K-major  bf16 STORE,ffn2" --groups 64 --rows 1024 --cublas
