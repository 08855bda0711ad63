#!/bin/bash
# Round-1 session-4 check + profile pass: GPU tests, default bench, launch list of the
# default bench command, ncu --set full captures of the cfg2/cfg3 top kernels (each ncu
# command runs only after the same command exited 0 without ncu).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
NCU="ncu --set full --import-source on --clock-control none"
REP=/tmp/ncu_reps; mkdir -p $REP
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/d_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/d_pytest.log
timeout 900 python bench.py > gpurun_out/d_bench_cfg2.log 2>&1; echo "bench rc=$?"
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-full-eval > gpurun_out/d_p4.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv --log-file gpurun_out/d_cfg2_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-full-eval > gpurun_out/d_n4.log 2>&1
python tools/probe_cfg.py cfg2 200000 > gpurun_out/d_p1.log 2>&1 && \
  timeout 900 $NCU -k regex:"k_dist_tile|k_resolve2|k_plan|k_chain2" --launch-skip 600 -c 8 -o $REP/d_cfg2_k1k3 python tools/probe_cfg.py cfg2 200000 > gpurun_out/d_n1.log 2>&1
python tools/probe_cfg.py cfg3 60000 > gpurun_out/d_p2.log 2>&1 && \
  timeout 900 $NCU -k regex:"k_tc_dots|k_resolve3|k_chain2|k_gram" --launch-skip 150 -c 8 -o $REP/d_cfg3_k1k3 python tools/probe_cfg.py cfg3 60000 > gpurun_out/d_n2.log 2>&1
for r in $REP/*.ncu-rep; do python tools/ncu_summary.py $r > gpurun_out/$(basename $r .ncu-rep)_summary.txt 2>&1; done
python tools/launch_summary.py gpurun_out/d_cfg2_launches.csv 40 > gpurun_out/d_cfg2_launches_summary.txt 2>&1
gzip -f gpurun_out/d_cfg2_launches.csv
du -sh gpurun_out
echo done
