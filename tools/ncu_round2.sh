# ncu --set full captures of the round-2 hot kernels (one GPU, one process each;
# every command first ran clean without ncu in the same session):
#   cfg2 (200k-row prefix): K1 chain walk, k_plan, K3 resolve, panel publication
#   cfg4 (one 1.46M-row shard): the tcgen05 panel contraction and its splits
#   cfg3 piece projection: the DMMA GEMM, blocked Cholesky, Jacobi
#   cfg2 clustering: seeding, batched Lloyd assignment, Lloyd tail
set -x
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on"
T=${TAG:-r2n}
R=/tmp/ncu_reps; mkdir -p $R
python bench.py --ncu --rows 200000 > /dev/null 2>&1 && \
$N -k regex:"k_chain2|k_plan|k_resolve2|k_publish_panel" --launch-skip 300 --launch-count 8 -o $R/${T}_cfg2_k1k3 \
  python bench.py --ncu --rows 200000 > gpurun_out/${T}_ncu1.log 2>&1
python bench.py --ncu --config cfg4 --rows 1460000 > /dev/null 2>&1 && \
$N -k regex:"k_tc_dots|k_tc_split|k_chain2" --launch-skip 600 --launch-count 6 -o $R/${T}_cfg4_panel \
  python bench.py --ncu --config cfg4 --rows 1460000 > gpurun_out/${T}_ncu2.log 2>&1
$N -k regex:"k_gemm|k_chol_blk|k_jacobi" --launch-count 10 -o $R/${T}_cfg3_proj python tools/probe_rsvd.py cfg3 --ncu > gpurun_out/${T}_ncu3.log 2>&1
$N -k regex:"k_seed_coop|k_lloyd_tail|k_update" --launch-count 6 -o $R/${T}_cfg2_kmeans \
  python bench.py --ncu --rows 200000 > gpurun_out/${T}_ncu4.log 2>&1
for f in $R/${T}_*.ncu-rep; do python tools/ncu_summary.py $f > gpurun_out/$(basename $f .ncu-rep)_summary.txt 2>&1; done
ls -la $R gpurun_out/${T}_*
