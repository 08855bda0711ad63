# Build with the device timeline stamps, run one cfg2 step, bring the phase means back.
set -x
mkdir -p gpurun_out
PCY_NVCC_EXTRA=-DPCY_TIMELINE python -m paper_1502_04265_b200._build --force > /dev/null 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-full-eval ${BARGS} > gpurun_out/timeline_bench.json 2> gpurun_out/timeline.err
grep "^\[timeline" gpurun_out/timeline.err | tail -6 | tr '|' '\n'
