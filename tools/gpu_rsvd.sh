mkdir -p gpurun_out
for c in cfg1 cfg3 cfg5; do python tools/probe_rsvd.py $c; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_rsvd_cfg1.csv python tools/probe_rsvd.py cfg1 --ncu > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_rsvd_cfg3.csv python tools/probe_rsvd.py cfg3 --ncu > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${TAG}_rsvd_cfg1.csv | head -20
python tools/launch_summary.py gpurun_out/${TAG}_rsvd_cfg3.csv | head -20
