set -x
mkdir -p gpurun_out
PCY_NVCC_EXTRA=-DPCY_TRACE python -m paper_1502_04265_b200._build --force > /dev/null 2>&1
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-full-eval > gpurun_out/trace_bench.json 2> gpurun_out/trace.err
grep -c "^\[ins\]" gpurun_out/trace.err
grep "^\[ins\]\|^\[rea\]" gpurun_out/trace.err | gzip > gpurun_out/trace_windows.txt.gz
rm gpurun_out/trace.err
