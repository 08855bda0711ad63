set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-full-eval"
$B > gpurun_out/ab1_cfg2_base.json 2>gpurun_out/ab1_err1.txt
PCY_NO_FULLSET=1 $B > gpurun_out/ab1_cfg2_nofs.json 2>>gpurun_out/ab1_err1.txt
B4="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-full-eval --config cfg4"
$B4 > gpurun_out/ab1_cfg4_base.json 2>>gpurun_out/ab1_err1.txt
PCY_NO_FULLSET=1 $B4 > gpurun_out/ab1_cfg4_nofs.json 2>>gpurun_out/ab1_err1.txt
B3="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-full-eval --config cfg3"
$B3 > gpurun_out/ab1_cfg3_base.json 2>>gpurun_out/ab1_err1.txt
PCY_NO_FULLSET=1 $B3 > gpurun_out/ab1_cfg3_nofs.json 2>>gpurun_out/ab1_err1.txt
tail -3 gpurun_out/ab1_err1.txt
