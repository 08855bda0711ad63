# ncu --set full capture of late k_resolve2x windows (cfg2 prefix); source page with CUDA-C correlation.
set -x
mkdir -p gpurun_out
T=${TAG:-r2ae}
R=/tmp/ncu_reps; mkdir -p $R
python bench.py --ncu --rows 200000 > gpurun_out/${T}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KERN:-k_resolve2x}" --launch-skip ${SKIP:-150} --launch-count ${COUNT:-2} -o $R/${T}_k -f \
  python bench.py --ncu --rows 200000 > gpurun_out/${T}_ncu1.log 2>&1
ncu -i $R/${T}_k.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/${T}_raw.csv.gz
ncu -i $R/${T}_k.ncu-rep --page source --print-source cuda,sass --csv 2>/dev/null | gzip > gpurun_out/${T}_source.csv.gz
ls -la gpurun_out/${T}_*
