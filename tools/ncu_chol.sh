ncu --set full -k regex:k_chol_blk -c 1 --import-source on -o gpurun_out/chol_blk python tools/probe_rsvd.py cfg1 --ncu > /dev/null 2>&1
ncu -i gpurun_out/chol_blk.ncu-rep --page details --csv 2>/dev/null | grep -E "Duration|Warp Cycles Per Issued|Stall|Issued Ipc|Achieved Occupancy|Registers" | head -30
