# r01j profile set of `bench.py` (C3): launch list + ncu --set full of the kNN8 walk phase
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/bench_short.json 2>&1 || { echo "bench failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01j.csv $CMD > gpurun_out/ncu_launches_r01j.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:'_ZN3fkd11walk_kernelILi3ELi4ELi8ELb0ELb0E|_ZN3fkd17walk_round_kernelILi3ELi4ELi8E|_ZN3fkd15overflow_kernelILi3ELi4ELi8E' \
    -c 6 -o gpurun_out/prof_knn8_r01j $CMD > gpurun_out/ncu_knn8_r01j.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_knn8_r01j.ncu-rep > gpurun_out/r01j_knn8_kernels.jsonl
python tools/launch_table.py gpurun_out/launches_r01j.csv "r01j launch list: bench.py --steps 2 --warmup 3 --no-cpu-baseline (C3, final kernels)" > gpurun_out/r01j_bench_launches.md
head -12 gpurun_out/r01j_bench_launches.md
