# Round-2 measurement set on the GPU box: GPU suite + smoke, the default bench
# line (cfg2, full contract incl. the CPU baseline), the reference arm, the
# other configs' bench lines, and the launch list of the default bench command
# (each ncu command only after the same command exited 0 without ncu).
set -x
mkdir -p gpurun_out
T=${TAG:-r2m}
timeout 1800 python -m pytest tests -m gpu -q -rfE > gpurun_out/${T}_pytest.txt 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/${T}_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/${T}_smoke.txt
timeout 900 python bench.py > gpurun_out/${T}_bench_cfg2.json 2> gpurun_out/${T}_bench_cfg2.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/${T}_bench_reference_cfg2.json 2> gpurun_out/${T}_bench_reference.err; echo "ref rc=$?"
for c in ${CFGS:-cfg1 cfg3 cfg4 cfg5}; do
  timeout 1500 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err; echo "$c rc=$?"
done
if [ -n "${LAUNCHES:-1}" ]; then
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_cfg2_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-full-eval > gpurun_out/${T}_ncu_launch.log 2>&1
  python tools/launch_summary.py gpurun_out/${T}_cfg2_launches.csv > gpurun_out/${T}_cfg2_launches_summary.txt 2>&1
  gzip -f gpurun_out/${T}_cfg2_launches.csv
fi
