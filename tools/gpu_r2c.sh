set -x
mkdir -p gpurun_out
python tools/repro_proj2.py 2>&1 | tail -9
python tools/repro_c6.py 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q -rfE > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/${TAG}_pytest.txt
bash tools/run_ref_tests.sh run
