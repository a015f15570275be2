# Round-end profile set of `bench.py` (C3): launch list + ncu --set full of the kNN8 and fcp walk phases
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/bench_short.json 2>&1 || { echo "bench failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01i.csv $CMD > gpurun_out/ncu_launches_r01i.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:'_ZN3fkd11walk_kernelILi3ELi4ELi8ELb0ELb0E|_ZN3fkd17walk_round_kernelILi3ELi4ELi8E|_ZN3fkd15overflow_kernelILi3ELi4ELi8E' \
    -c 6 -o gpurun_out/prof_knn8_r01i $CMD > gpurun_out/ncu_knn8_r01i.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:'_ZN3fkd11walk_kernelILi3ELi4ELi1ELb0ELb0E|_ZN3fkd17walk_round_kernelILi3ELi4ELi1E|_ZN3fkd15overflow_kernelILi3ELi4ELi1E' \
    -c 6 -o gpurun_out/prof_fcp_r01i $CMD > gpurun_out/ncu_fcp_r01i.log 2>&1
tail -1 gpurun_out/ncu_knn8_r01i.log; tail -1 gpurun_out/ncu_fcp_r01i.log
python tools/ncu_summary.py gpurun_out/prof_knn8_r01i.ncu-rep > gpurun_out/r01i_knn8_kernels.jsonl
python tools/ncu_summary.py gpurun_out/prof_fcp_r01i.ncu-rep > gpurun_out/r01i_fcp_kernels.jsonl
python tools/launch_table.py gpurun_out/launches_r01i.csv "r01i launch list: bench.py --steps 2 --warmup 3 --no-cpu-baseline (C3, final kernels)" > gpurun_out/r01i_bench_launches.md
head -12 gpurun_out/r01i_bench_launches.md
