# One bench line per config given in $CFGS (default cfg2), full bench (cpu baseline included).
set -x
mkdir -p gpurun_out
for c in ${CFGS:-cfg2}; do
  python bench.py --config $c ${BARGS:---steps 5 --warmup 3} > gpurun_out/${TAG}_bench_$c.json 2>gpurun_out/${TAG}_bench_$c.err
  tail -2 gpurun_out/${TAG}_bench_$c.err
done
