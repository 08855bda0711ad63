#!/bin/bash
# launch list of the k-means phases on a cfg5-shaped coreset (debug)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/km_launches.csv \
  python tools/probe_kmeans.py 25000 4096 250 5 100 > gpurun_out/km_ncu.log 2>&1
