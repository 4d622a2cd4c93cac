cd $GRAFT_REPO_ROOT
timeout 120 python benchmarks/gather_bench.py --only c2,c3,c4
timeout 120 python benchmarks/gather_bench.py --only c2,c4 --seq
timeout 300 ncu --set full --import-source on --clock-control none -k regex:tc_gemm -s 3 -c 1 -o gpurun_out/gather_c4 -f python benchmarks/gather_bench.py --only c4 --reps 1 > gpurun_out/gather_ncu.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:tc_gemm -s 3 -c 1 -o gpurun_out/gather_c2 -f python benchmarks/gather_bench.py --only c2 --reps 1 >> gpurun_out/gather_ncu.log 2>&1
