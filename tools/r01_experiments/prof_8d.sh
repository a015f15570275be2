# ncu --set full of the 8-D kNN16 first walk and resume pass (C4-8D, M=1M)
CMD="python tools/quickbench.py --dim 8 --m 1000000 --configs knn16 --reps 1 --sorted-only"
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:'_ZN3fkd11walk_kernelILi8ELi8ELi16ELb0ELb0E|_ZN3fkd17walk_round_kernelILi8ELi8ELi16E' \
    -c 2 -o gpurun_out/prof_8d $CMD > gpurun_out/ncu_8d.log 2>&1
tail -2 gpurun_out/ncu_8d.log
python tools/ncu_summary.py gpurun_out/prof_8d.ncu-rep > gpurun_out/r01i_8d_kernels.jsonl
cat gpurun_out/r01i_8d_kernels.jsonl
