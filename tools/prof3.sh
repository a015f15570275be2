export FKD_QPL=8
python tools/quickbench.py --configs fcp --reps 1 > gpurun_out/p_q8.log 2>&1 && \
ncu --set full --clock-control none --kernel-name-base mangled -k regex:walk_multi -s 1 -c 1 -o gpurun_out/prof_multi_fcp python tools/quickbench.py --configs fcp --reps 1 > gpurun_out/ncu_q8.log 2>&1
tail -1 gpurun_out/ncu_q8.log
