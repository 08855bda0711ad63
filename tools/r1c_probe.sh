#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
PCY_DEBUG_REBUILD=1 PCY_TRACE_K3=gpurun_out/p_trace_cfg2.txt timeout 600 python tools/probe_cfg.py cfg2 581012 > gpurun_out/p_cfg2.log 2>&1; echo "cfg2 rc=$?"
PCY_DEBUG_REBUILD=1 PCY_TRACE_K3=gpurun_out/p_trace_cfg3.txt timeout 600 python tools/probe_cfg.py cfg3 200000 > gpurun_out/p_cfg3.log 2>&1; echo "cfg3 rc=$?"
PCY_DEBUG_REBUILD=1 PCY_TRACE_K3=gpurun_out/p_trace_cfg5.txt timeout 600 python tools/probe_cfg.py cfg5 125000 > gpurun_out/p_cfg5.log 2>&1; echo "cfg5 rc=$?"
gzip -f gpurun_out/p_trace_*.txt
