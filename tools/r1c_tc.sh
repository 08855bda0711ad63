#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
PCY_TC_PARTS=1 timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/t_pytest.log 2>&1; echo "pytest tc rc=$?"; tail -3 gpurun_out/t_pytest.log
PCY_TC_PARTS=1 PCY_TRACE_K3=gpurun_out/t_trace_cfg2.txt timeout 600 python tools/probe_cfg.py cfg2 581012 > gpurun_out/t_cfg2.log 2>&1; echo "cfg2 rc=$?"
PCY_TC_PARTS=1 PCY_TRACE_K3=gpurun_out/t_trace_cfg1.txt timeout 600 python tools/probe_cfg.py cfg1 20000 > gpurun_out/t_cfg1.log 2>&1; echo "cfg1 rc=$?"
timeout 600 python tools/probe_cfg.py cfg1 20000 > gpurun_out/t_cfg1_dmma.log 2>&1; echo "cfg1 rc=$?"
PCY_TC_PARTS=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/t_bench_cfg2.log 2>&1; echo "bench rc=$?"
gzip -f gpurun_out/t_trace_*.txt
