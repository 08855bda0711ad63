#!/bin/bash
# Round-1 final measurements: bench lines for every config, the reference arm,
# the launch list of the default bench command and ncu --set full captures of
# the top kernels (each ncu command runs only after the same command exited 0).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
NCU="ncu --set full --import-source on --clock-control none"
REP=/tmp/ncu_reps; mkdir -p $REP
timeout 900 python bench.py > gpurun_out/f_bench_cfg2.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/f_bench_ref.log 2>&1; echo "ref rc=$?"
for c in cfg1 cfg3 cfg4 cfg5; do
  timeout 1500 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/f_bench_$c.log 2>&1
  echo "$c rc=$?"
done
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-full-eval > gpurun_out/f_p4.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv --log-file gpurun_out/f_cfg2_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-full-eval > gpurun_out/f_n4.log 2>&1
python tools/probe_cfg.py cfg2 200000 > gpurun_out/f_p1.log 2>&1 && \
  timeout 900 $NCU -k regex:"k_dist_tile|k_resolve2|k_plan" --launch-skip 600 -c 6 -o $REP/f_cfg2_k1k3 python tools/probe_cfg.py cfg2 200000 > gpurun_out/f_n1.log 2>&1
python tools/probe_cfg.py cfg3 60000 > gpurun_out/f_p2.log 2>&1 && \
  timeout 900 $NCU -k regex:"k_tc_dots|k_resolve3|k_chain2" --launch-skip 150 -c 6 -o $REP/f_cfg3_k1k3 python tools/probe_cfg.py cfg3 60000 > gpurun_out/f_n2.log 2>&1
python tools/probe_kmeans.py 25000 4096 250 5 20 > gpurun_out/f_p3.log 2>&1 && \
  timeout 900 $NCU -k regex:k_seed_coop -c 1 -o $REP/f_seed python tools/probe_kmeans.py 25000 4096 250 5 20 > gpurun_out/f_n3.log 2>&1
for r in $REP/*.ncu-rep; do python tools/ncu_summary.py $r > gpurun_out/$(basename $r .ncu-rep)_summary.txt 2>&1; done
python tools/launch_summary.py gpurun_out/f_cfg2_launches.csv 40 > gpurun_out/f_cfg2_launches_summary.txt 2>&1
gzip -f gpurun_out/f_cfg2_launches.csv
du -sh gpurun_out
echo done
