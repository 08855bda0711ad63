set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rfE > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/${TAG}_pytest.txt
for c in cfg2 cfg1 cfg3; do
  python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-full-eval > gpurun_out/${TAG}_$c.json 2>gpurun_out/${TAG}_$c.err; tail -2 gpurun_out/${TAG}_$c.err
done
