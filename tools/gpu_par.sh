cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_engine_gpu.py tests/test_golden_gpu.py -x -q > gpurun_out/t_engine.log 2>&1; echo "rc=$?" >> gpurun_out/t_engine.log
PCY_TRACE_K3=gpurun_out/trace_par.txt timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-full-eval > gpurun_out/bench_par_trace.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-full-eval > gpurun_out/bench_par.log 2>&1
