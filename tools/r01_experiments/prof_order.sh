# ncu of the Morton ordering kernels (counting sort) in the C3 bench step
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
ncu --set full --clock-control none -k regex:'morton_rank|morton_scatter' -c 4 -o gpurun_out/prof_order $CMD > gpurun_out/ncu_order.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_order.ncu-rep > gpurun_out/order_kernels.jsonl
