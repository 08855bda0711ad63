#!/bin/bash
# Round-1 session-4 final measurements: bench lines (all configs + reference arm), launch list
# of the default bench command, ncu --set full key metrics of the cfg2/cfg3 top kernels.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
NCU="ncu --set full --import-source on --clock-control none"
REP=/tmp/ncu_f; rm -rf $REP; mkdir -p $REP
timeout 900 python bench.py > gpurun_out/r1f_bench_cfg2.log 2>&1; echo "cfg2 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r1f_bench_ref.log 2>&1; echo "ref rc=$?"
for c in cfg1 cfg3 cfg4 cfg5; do
  timeout 1500 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1f_bench_$c.log 2>&1; echo "$c rc=$?"
done
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-full-eval > gpurun_out/f_p4.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv --log-file gpurun_out/r1f_cfg2_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-full-eval > gpurun_out/f_n4.log 2>&1; echo "launches rc=$?"
python tools/probe_cfg.py cfg2 581012 > gpurun_out/f_p1.log 2>&1 && \
  timeout 900 $NCU -k regex:"k_dist_tile|k_resolve2|k_plan|k_chain2|k_reattach2" --launch-skip 3000 -c 10 -o $REP/r1f_cfg2 python tools/probe_cfg.py cfg2 581012 > gpurun_out/f_n1.log 2>&1; echo "ncu cfg2 rc=$?"
python tools/probe_cfg.py cfg3 60000 > gpurun_out/f_p2.log 2>&1 && \
  timeout 900 $NCU -k regex:"k_tc_dots|k_resolve3|k_chain2" --launch-skip 150 -c 6 -o $REP/r1f_cfg3 python tools/probe_cfg.py cfg3 60000 > gpurun_out/f_n2.log 2>&1; echo "ncu cfg3 rc=$?"
for r in $REP/*.ncu-rep; do python tools/ncu_summary.py $r > gpurun_out/$(basename $r .ncu-rep)_summary.txt 2>&1; done
python tools/launch_summary.py gpurun_out/r1f_cfg2_launches.csv 40 > gpurun_out/r1f_cfg2_launches_summary.txt 2>&1
gzip -f gpurun_out/r1f_cfg2_launches.csv
du -sh gpurun_out
echo done
