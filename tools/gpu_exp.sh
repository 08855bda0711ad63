cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PCY_NO_FULLSET=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-full-eval > gpurun_out/bench_nofs.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/launches_nofs.csv env PCY_NO_FULLSET=1 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-full-eval --ncu > gpurun_out/ncu_nofs.log 2>&1
