set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_linalg_gpu.py tests/test_pipeline_gpu.py tests/test_mergereduce_gpu.py tests/test_golden_gpu.py "tests/test_fullsize_gpu.py::test_full_config_matches_reference[cfg1]" "tests/test_fullsize_gpu.py::test_full_config_matches_reference[cfg3]" -q -x -rfE > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/${TAG}_pytest.txt
for c in cfg1 cfg3 cfg5; do timeout 300 python tools/probe_rsvd.py $c; done
for c in cfg1 cfg3; do ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_rsvd_$c.csv python tools/probe_rsvd.py $c --ncu > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/${TAG}_rsvd_$c.csv | head -14; done
