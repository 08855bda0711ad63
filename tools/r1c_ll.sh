#!/bin/bash
# launch list (per-kernel durations) of the single-shard cfg5 probe and the cfg3 probe
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for c in "cfg5 125000" "cfg3 200000"; do
  set -- $c
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60000 --csv --log-file gpurun_out/ll_$1.csv \
    python tools/probe_cfg.py $1 $2 > gpurun_out/ll_$1.log 2>&1; echo "$1 rc=$?"
  python tools/launch_summary.py gpurun_out/ll_$1.csv 30 > gpurun_out/ll_$1_summary.txt 2>&1
  gzip -f gpurun_out/ll_$1.csv
done
