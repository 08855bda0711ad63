#!/bin/bash
# Round-1 session-4 bench lines (timed steps un-instrumented; per-kernel breakdown from a second pass).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r1e_bench_cfg2.log 2>&1; echo "cfg2 rc=$?"; tail -1 gpurun_out/r1e_bench_cfg2.log | cut -c1-400
timeout 900 python bench.py --impl reference > gpurun_out/r1e_bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/r1e_bench_ref.log | cut -c1-300
for c in ${CONFIGS:-cfg1 cfg3}; do
  timeout 1500 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1e_bench_$c.log 2>&1; echo "$c rc=$?"; tail -1 gpurun_out/r1e_bench_$c.log | cut -c1-300
done
echo done
