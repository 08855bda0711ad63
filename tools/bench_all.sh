#!/bin/bash
# One short bench line per config (for DESIGN.md / profiles); not the driver's bench.
mkdir -p gpurun_out
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 1500 python bench.py --config $c --steps ${STEPS:-1} --warmup ${WARMUP:-1} --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
  tail -1 gpurun_out/bench_$c.log > gpurun_out/bench_$c.json
  echo "$c rc=$?"
done
