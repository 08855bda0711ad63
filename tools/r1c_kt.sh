#!/bin/bash
# per-kernel durations of selected kernels (cfg5 shard probe, k-means probe)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
tag=${1:-kt}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_jacobi|k_dist_tile|k_tc_dots|k_chain2|k_resolve3|k_plan" -c 3000 --csv --log-file gpurun_out/${tag}_cfg5.csv \
    python tools/probe_cfg.py cfg5 60000 > gpurun_out/${tag}_cfg5.log 2>&1; echo "cfg5 rc=$?"
python tools/launch_summary.py gpurun_out/${tag}_cfg5.csv 30 > gpurun_out/${tag}_cfg5_summary.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_seed_coop" -c 2 --csv --log-file gpurun_out/${tag}_seed.csv \
    python tools/probe_kmeans.py 25000 4096 250 5 20 > gpurun_out/${tag}_seed.log 2>&1; echo "seed rc=$?"
gzip -f gpurun_out/${tag}_cfg5.csv
