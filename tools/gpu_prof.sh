cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PCY_TRACE_K3=gpurun_out/trace_cfg2.txt timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-full-eval > gpurun_out/b_tr2.log 2>&1
PCY_TRACE_K3=gpurun_out/trace_cfg3.txt timeout 600 python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline --no-full-eval > gpurun_out/b_tr3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-full-eval --ncu > gpurun_out/ncu_cfg2.log 2>&1
