cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches_cfg3.csv python bench.py --config cfg3 --rows 60000 --steps 1 --warmup 0 --no-cpu-baseline --no-full-eval --ncu > gpurun_out/ncu_cfg3.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_cfg3.log
