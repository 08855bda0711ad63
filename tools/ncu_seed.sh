# ncu --set full capture of the seeding kernel on the cfg3 coreset (source-level csv comes back)
set -x
mkdir -p gpurun_out
T=${TAG:-r2y}
R=/tmp/ncu_reps; mkdir -p $R
python bench.py --ncu --config ${CFG:-cfg3} > gpurun_out/${T}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_seed_coop" --launch-count 1 -o $R/${T}_seed -f \
  python bench.py --ncu --config ${CFG:-cfg3} > gpurun_out/${T}_ncu1.log 2>&1
for f in $R/${T}_*.ncu-rep; do
  b=$(basename $f .ncu-rep)
  ncu -i $f --page raw --csv 2>/dev/null | gzip > gpurun_out/${b}_raw.csv.gz
  ncu -i $f --page source --csv 2>/dev/null | gzip > gpurun_out/${b}_source.csv.gz
done
ls -la gpurun_out/${T}_*
