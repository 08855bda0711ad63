#!/bin/bash
# Check: GPU parity suite, cfg2/cfg3/cfg4 bench lines after the side-stream Gram and the sliced rebuild rank.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
J='import json,sys; l=json.loads(sys.stdin.readlines()[-1]); print(round(l["value"]), round(l["e2e"]["value"]), round(l["ms_per_step"],2), {k: round(v["ms"],2) for k,v in l["kernel_ms_per_step"].items()}, l["phase_ms"][-1])'
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in cfg2 cfg3; do
  echo "== $c"; timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-full-eval > gpurun_out/ab_$c.log 2>&1; tail -1 gpurun_out/ab_$c.log | python -c "$J"
done
echo "== cfg4"; timeout 900 python bench.py --config cfg4 --steps 2 --warmup 1 --no-cpu-baseline --no-full-eval > gpurun_out/ab_cfg4.log 2>&1; tail -1 gpurun_out/ab_cfg4.log | python -c "$J"
echo done
