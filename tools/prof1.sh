export FKD_PERSIST=0
python tools/quickbench.py --clustered --configs knn8 --reps 1 > gpurun_out/plain_knn8.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:walk_kernel -s 1 -c 1 -o gpurun_out/prof_knn8_clu python tools/quickbench.py --clustered --configs knn8 --reps 1 > gpurun_out/ncu_knn8.log 2>&1
python tools/quickbench.py --configs fcp --reps 1 > gpurun_out/plain_fcp.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:walk_kernel -s 1 -c 1 -o gpurun_out/prof_fcp_uni python tools/quickbench.py --configs fcp --reps 1 > gpurun_out/ncu_fcp.log 2>&1
ls -la gpurun_out
