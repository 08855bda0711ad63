#!/bin/bash
# Full GPU suite + cfg2/cfg3 bench lines after moving every DMMA tile kernel to cp.async staging.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
J='import json,sys; l=json.loads(sys.stdin.readlines()[-1]); print(round(l["value"]), round(l["e2e"]["value"]), round(l["ms_per_step"],2), {k: round(v["ms"],2) for k,v in l["kernel_ms_per_step"].items()}, [(r["kernel"][:14], round(r["ms_per_step"],2), round(r["frac"],3)) for r in l["rooflines"]], l["phase_ms"][-1])'
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in cfg2 cfg3 cfg2; do
  echo "== $c"; timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-full-eval > gpurun_out/ck_$c.log 2>&1; tail -1 gpurun_out/ck_$c.log | python -c "$J"

done
echo done
