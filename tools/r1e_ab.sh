#!/bin/bash
# A/B: cp.async double-buffered DMMA parts (k_dist_tile<2, true>) vs register-staged (PCY_OLD_PARTS=1).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
J='import json,sys; l=json.loads(sys.stdin.readlines()[-1]); print(round(l["value"]), round(l["ms_per_step"],2), {k: round(v["ms"],2) for k,v in l["kernel_ms_per_step"].items()}, [(r["kernel"][:14], round(r["ms_per_step"],2), round(r["frac"],3)) for r in l["rooflines"]][:1])'
timeout 1200 python -m pytest tests/test_engine_gpu.py tests/test_golden_gpu.py tests/test_pipeline_gpu.py tests/test_mergereduce_gpu.py -x -q 2>&1 | tail -2
for v in "" "PCY_OLD_PARTS=1" "" "PCY_OLD_PARTS=1"; do
  echo "== $v"; env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-full-eval > gpurun_out/ab.log 2>&1; tail -1 gpurun_out/ab.log | python -c "$J"
done
echo done
