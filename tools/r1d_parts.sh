#!/bin/bash
# k_parts_cp (cp.async-staged DMMA parts, K <= 64) against k_dist_tile<2>: parity tests,
# cfg2 bench with each kernel, ncu capture of the new kernel.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
REP=/tmp/ncu_reps; mkdir -p $REP
timeout 1200 python -m pytest tests/test_engine_gpu.py tests/test_golden_gpu.py tests/test_pipeline_gpu.py tests/test_mergereduce_gpu.py -x -q > gpurun_out/e_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/e_pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-full-eval > gpurun_out/e_bench_new.log 2>&1; echo "bench new rc=$?"
PCY_OLD_PARTS=1 timeout 600 python bench.py --no-cpu-baseline --no-full-eval > gpurun_out/e_bench_old.log 2>&1; echo "bench old rc=$?"
python tools/probe_cfg.py cfg2 200000 > gpurun_out/e_p1.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_parts_cp" --launch-skip 600 -c 3 -o $REP/e_parts python tools/probe_cfg.py cfg2 200000 > gpurun_out/e_n1.log 2>&1
PCY_DEBUG_REBUILD=1 timeout 300 python tools/probe_cfg.py cfg2 581012 > gpurun_out/e_rebuild.log 2>&1; echo "rebuild trace rc=$?"
for r in $REP/*.ncu-rep; do python tools/ncu_summary.py $r > gpurun_out/$(basename $r .ncu-rep)_summary.txt 2>&1; cp $r gpurun_out/; done
echo done
