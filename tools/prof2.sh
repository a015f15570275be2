export FKD_BUDGET=0
for r in 4 16; do
FKD_PERSIST=1 FKD_REFILL=$r python tools/quickbench.py --configs fcp --reps 1 > gpurun_out/p_$r.log 2>&1 && \
FKD_PERSIST=1 FKD_REFILL=$r ncu --set full --clock-control none -k regex:walk_persistent -s 1 -c 1 -o gpurun_out/prof_pers_fcp_r$r python tools/quickbench.py --configs fcp --reps 1 > gpurun_out/ncu_p$r.log 2>&1
done
ls gpurun_out
