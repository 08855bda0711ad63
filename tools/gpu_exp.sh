cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config cfg3 --steps 2 --warmup 1 --no-cpu-baseline --no-full-eval > gpurun_out/bench_cfg3.log 2>&1
python tools/probe_cfg.py cfg3 60000 > gpurun_out/x_p.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_resolve3" --launch-skip 80 -c 1 -o /tmp/r3 python tools/probe_cfg.py cfg3 60000 > gpurun_out/x_n.log 2>&1
ncu -i /tmp/r3.ncu-rep --page source --csv --print-source sass > gpurun_out/r3_sass.csv 2>/dev/null
ncu -i /tmp/r3.ncu-rep --page details --csv > gpurun_out/r3_details.csv 2>/dev/null
gzip -f gpurun_out/r3_sass.csv
du -sh gpurun_out
