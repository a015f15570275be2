# ncu --set full of the C3 kNN8 walk, its rounds and CTA pass in `bench.py`
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:'_ZN3fkd11walk_kernelILi3ELi4ELi8ELb0ELb0E|_ZN3fkd17walk_round_kernelILi3ELi4ELi8E|_ZN3fkd15overflow_kernelILi3ELi4ELi8E' \
    -c 6 -o gpurun_out/prof_knn8 $CMD > gpurun_out/ncu_knn8.log 2>&1
tail -2 gpurun_out/ncu_knn8.log
python tools/ncu_summary.py gpurun_out/prof_knn8.ncu-rep > gpurun_out/r01f_knn8_kernels.jsonl
