# A/B of the visited-groups K1: GPU suite, then cfg2 / cfg4 bench lines.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.txt
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-full-eval"
$B > gpurun_out/${TAG}_cfg2.json 2>gpurun_out/${TAG}_err.txt
$B --config cfg4 --steps 1 --warmup 1 > gpurun_out/${TAG}_cfg4.json 2>>gpurun_out/${TAG}_err.txt
tail -3 gpurun_out/${TAG}_err.txt
