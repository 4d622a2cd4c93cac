cd $GRAFT_REPO_ROOT
for v in rbold rbwarp; do
MOE_B200_LIB=exp/$v/libmoe_b200.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:route_bwd -s 2 -c 1 -o gpurun_out/rb_$v -f python bench.py --config c2 --steps 1 --warmup 1 --no-cpu --no-ring --no-e2e > gpurun_out/rbncu_$v.log 2>&1; echo $v rc=$?
done
