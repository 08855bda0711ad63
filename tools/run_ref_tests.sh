# Run the reference's own test suite (pkg/tests) against the drop-in through
# the `piecy` shim in tools/refshim.
#   here (build container):  bash tools/run_ref_tests.sh stage
#   on the GPU box:          bash tools/run_ref_tests.sh run
# `stage` copies /root/reference/pkg/tests into baseline/_ref_tests
# (git-ignored, never committed; it travels to the box with the snapshot).
set -u
case "${1:-run}" in
  stage)
    rm -rf baseline/_ref_tests && mkdir -p baseline/_ref_tests
    cp /root/reference/pkg/tests/*.py baseline/_ref_tests/
    ls baseline/_ref_tests ;;
  run)
    mkdir -p gpurun_out
    cd baseline/_ref_tests
    PYTHONPATH=$GRAFT_REPO_ROOT/tools/refshim:$PWD:$GRAFT_REPO_ROOT timeout 2400 python -m pytest . -p no:cacheprovider \
      -q -rfE --durations=10 -o addopts="" --rootdir . > $GRAFT_REPO_ROOT/gpurun_out/${TAG:-r2}_reftests.txt 2>&1
    echo "reftests rc=$?"
    tail -30 $GRAFT_REPO_ROOT/gpurun_out/${TAG:-r2}_reftests.txt ;;
esac
