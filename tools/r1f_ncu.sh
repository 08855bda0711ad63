#!/bin/bash
# Session-5 ncu --set full capture of the cfg2 K1/K3 kernels after the cp.async DMMA tiles
# and the Gram-scored reattach table (probe run first; ncu only after it exited 0).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
NCU="ncu --set full --import-source on --clock-control none"
REP=/tmp/ncu_g; rm -rf $REP; mkdir -p $REP
timeout 300 python tools/probe_cfg.py cfg2 200000 > gpurun_out/g_p1.log 2>&1 && \
  timeout 700 $NCU -k regex:"k_dist_tile|k_resolve2|k_plan" --launch-skip 600 -c 6 -o $REP/r1f_cfg2_k1k3 python tools/probe_cfg.py cfg2 200000 > gpurun_out/g_n1.log 2>&1; echo "ncu rc=$?"
for r in $REP/*.ncu-rep; do python tools/ncu_summary.py $r > gpurun_out/$(basename $r .ncu-rep)_summary.txt 2>&1; done
echo done
