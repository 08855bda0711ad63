#!/bin/bash
# k_reattach2 with Gram dots for same-launch entries and a 320-entry table, vs reference rows (PCY_REA_TROWS=1).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
J='import json,sys; l=json.loads(sys.stdin.readlines()[-1]); print(round(l["value"]), round(l["e2e"]["value"]), round(l["ms_per_step"],2), {k: round(v["ms"],2) for k,v in l["kernel_ms_per_step"].items()}, l["phase_ms"][-1])'
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in "" "PCY_REA_TROWS=1" ""; do
  echo "== cfg2 $v"; env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-full-eval > gpurun_out/rea.log 2>&1; tail -1 gpurun_out/rea.log | python -c "$J"
done
echo "== cfg4"; timeout 900 python bench.py --config cfg4 --steps 2 --warmup 1 --no-cpu-baseline --no-full-eval > gpurun_out/rea4.log 2>&1; tail -1 gpurun_out/rea4.log | python -c "$J"
PCY_DEBUG_REBUILD=1 timeout 300 python tools/probe_cfg.py cfg2 581012 > gpurun_out/g_rebuild.log 2>&1; echo "rebuild trace rc=$?"; grep -c "reattach launch" gpurun_out/g_rebuild.log
echo done
