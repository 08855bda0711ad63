# GPU suite on the box: every -m gpu test (full-size parity included), then smoke().
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
free -g | head -2
timeout 3000 python -m pytest tests -m gpu -q -rA -x --durations=15 > gpurun_out/${TAG:-r2}_pytest_gpu.txt 2>&1
echo "pytest rc=$?"
tail -40 gpurun_out/${TAG:-r2}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG:-r2}_smoke.txt 2>&1
echo "smoke rc=$?"; tail -3 gpurun_out/${TAG:-r2}_smoke.txt
