set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -rfE > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/${TAG}_pytest.txt
bash tools/run_ref_tests.sh run
