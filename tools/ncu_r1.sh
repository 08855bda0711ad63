#!/bin/bash
# Round-1 ncu captures (one tool: ncu).  Each command first runs plainly (&&).
mkdir -p gpurun_out
NCU="ncu --set full --import-source on --clock-control none"
python tools/probe_cfg.py cfg3 60000 > gpurun_out/p1.log 2>&1 && \
  $NCU -k regex:k_tc_dots --launch-skip 60 -c 1 -o gpurun_out/r1_tc_dots python tools/probe_cfg.py cfg3 60000 > gpurun_out/n1.log 2>&1
python tools/probe_kmeans.py 17500 1024 100 5 100 > gpurun_out/p2.log 2>&1 && \
  $NCU -k regex:k_seed_coop -c 1 -o gpurun_out/r1_seed python tools/probe_kmeans.py 17500 1024 100 5 100 > gpurun_out/n2.log 2>&1
python tools/probe_cfg.py cfg2 200000 > gpurun_out/p3.log 2>&1 && \
  $NCU -k regex:"k_dist_tile|k_resolve2" --launch-skip 200 -c 2 -o gpurun_out/r1_cfg2_k1k3 python tools/probe_cfg.py cfg2 200000 > gpurun_out/n3.log 2>&1
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/p4.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r1_bench_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/n4.log 2>&1
echo done
