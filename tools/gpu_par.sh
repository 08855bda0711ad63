cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-full-eval > gpurun_out/bench_par.log 2>&1
timeout 900 python bench.py --config cfg3 --steps 2 --warmup 1 --no-cpu-baseline --no-full-eval > gpurun_out/bench_cfg3.log 2>&1
