cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none --csv --log-file gpurun_out/c4_launches.csv python bench.py --config c4 --steps 1 --warmup 1 --no-cpu --no-ring --no-e2e > gpurun_out/c4_ncu.log 2>&1
echo rc=$?
