#!/bin/bash
# A/B of the session-4 K1 changes on cfg2 (bench lines to stdout), rebuild trace, parts ncu summary.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
REP=/tmp/ncu_reps; mkdir -p $REP
B="python bench.py --no-cpu-baseline --no-full-eval"
J='import json,sys; l=json.loads(sys.stdin.readlines()[-1]); print(round(l["value"]), round(l["ms_per_step"],2), {k: round(v["ms"],2) for k,v in l["kernel_ms_per_step"].items()}, [(r["kernel"][:14], round(r["ms_per_step"],2), round(r["frac"],3)) for r in l["rooflines"]+[l["roofline"]]])'
timeout 1200 python -m pytest tests/test_engine_gpu.py tests/test_golden_gpu.py tests/test_pipeline_gpu.py tests/test_mergereduce_gpu.py tests/test_engine_highdim_gpu.py -x -q 2>&1 | tail -2
for v in "" "PCY_OLD_PARTS=1" "PCY_GRAM_LATE=1" "PCY_OLD_PARTS=1 PCY_GRAM_LATE=1" ""; do
  echo "== $v"; env $v timeout 600 $B > gpurun_out/ab.log 2>&1; tail -1 gpurun_out/ab.log | python -c "$J"
done
PCY_DEBUG_REBUILD=1 timeout 300 python tools/probe_cfg.py cfg2 581012 > gpurun_out/f_rebuild.log 2>&1; echo "rebuild trace rc=$?"
python tools/probe_cfg.py cfg2 200000 > gpurun_out/f_p1.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_parts_cp" --launch-skip 600 -c 3 -o $REP/f_parts python tools/probe_cfg.py cfg2 200000 > gpurun_out/f_n1.log 2>&1
echo "ncu rc=$?"
for r in $REP/*.ncu-rep; do python tools/ncu_summary.py $r > gpurun_out/$(basename $r .ncu-rep)_summary.txt 2>&1; done
du -sh gpurun_out
echo done
