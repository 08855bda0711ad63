# ncu --set full source-level capture of the rebuild reattach kernel (cfg2 prefix):
# the first window of a rebuild (one CTA, every node opens) and later K3 windows.
# The reports stay on the box; their raw and source pages come back as csv.gz.
set -x
mkdir -p gpurun_out
T=${TAG:-r2v}
R=/tmp/ncu_reps; mkdir -p $R
python bench.py --ncu --rows 200000 > gpurun_out/${T}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_reattach2x" --launch-count 2 -o $R/${T}_reattach_first -f \
  python bench.py --ncu --rows 200000 > gpurun_out/${T}_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_reattach2x|k_resolve2x" --launch-skip 230 --launch-count 3 -o $R/${T}_k3_late -f \
  python bench.py --ncu --rows 200000 > gpurun_out/${T}_ncu2.log 2>&1
for f in $R/${T}_*.ncu-rep; do
  b=$(basename $f .ncu-rep)
  ncu -i $f --page raw --csv 2>/dev/null | gzip > gpurun_out/${b}_raw.csv.gz
  ncu -i $f --page source --csv 2>/dev/null | gzip > gpurun_out/${b}_source.csv.gz
done
ls -la gpurun_out/${T}_*
