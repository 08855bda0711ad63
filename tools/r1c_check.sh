#!/bin/bash
# Session-3 check: GPU test suite, then bench lines for the default config and cfg3/cfg5.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/c_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/c_pytest.log
timeout 900 python bench.py > gpurun_out/c_bench_cfg2.log 2>&1; echo "bench rc=$?"
for c in cfg3 cfg5; do
  timeout 1200 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/c_bench_$c.log 2>&1
  echo "$c rc=$?"
done
echo done
