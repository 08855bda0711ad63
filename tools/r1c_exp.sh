#!/bin/bash
# experiment: GPU tests, then per-config probes with the K3 trace and rebuild log
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
tag=${1:-e}
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${tag}_pytest.log
for c in "cfg2 581012" "cfg1 20000" "cfg3 200000" "cfg5 125000"; do
  set -- $c
  PCY_DEBUG_REBUILD=1 PCY_TRACE_K3=gpurun_out/${tag}_trace_$1.txt timeout 600 python tools/probe_cfg.py $1 $2 > gpurun_out/${tag}_$1.log 2>&1; echo "$1 rc=$?"
  grep -v "reattach launch" gpurun_out/${tag}_$1.log | tail -3
done
timeout 300 python tools/probe_kmeans.py 25000 4096 250 5 20 > gpurun_out/${tag}_km.log 2>&1; echo "km rc=$?"; tail -4 gpurun_out/${tag}_km.log
gzip -f gpurun_out/${tag}_trace_*.txt
