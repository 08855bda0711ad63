set -x
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on"
T=r2z
R=/tmp/ncu_reps; mkdir -p $R
python bench.py --ncu --rows 200000 > /dev/null 2>&1 && \
$N -k regex:"k_chain2|k_plan|k_resolve2|k_reattach2" --launch-skip 300 --launch-count 12 -o $R/${T}_cfg2_k1k3 -f \
  python bench.py --ncu --rows 200000 > gpurun_out/${T}_ncu1.log 2>&1
python tools/ncu_summary.py $R/${T}_cfg2_k1k3.ncu-rep > gpurun_out/${T}_cfg2_k1k3_summary.txt 2>&1
