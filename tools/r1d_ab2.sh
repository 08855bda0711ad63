#!/bin/bash
# A/B: batch Gram on the side stream (live + rebuild) vs in line (PCY_GRAM_LATE=1).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
J='import json,sys; l=json.loads(sys.stdin.readlines()[-1]); print(round(l["value"]), round(l["e2e"]["value"]), round(l["ms_per_step"],2), {k: round(v["ms"],2) for k,v in l["kernel_ms_per_step"].items()}, l["phase_ms"][-1])'
timeout 1200 python -m pytest tests/test_engine_gpu.py tests/test_golden_gpu.py tests/test_pipeline_gpu.py tests/test_mergereduce_gpu.py tests/test_engine_highdim_gpu.py tests/test_tc_gpu.py -x -q 2>&1 | tail -2
for c in cfg2 cfg3; do
for v in "" "PCY_GRAM_LATE=1"; do
  echo "== $c $v"; env $v timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-full-eval > gpurun_out/ab_$c.log 2>&1; tail -1 gpurun_out/ab_$c.log | python -c "$J"
done; done
echo done
