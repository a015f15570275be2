# round profile: launch list + full captures of the dominant kernels of `bench.py`
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
    -k regex:'_ZN3fkd11walk_kernelILi3ELi4ELi8ELb0ELb0E|_ZN3fkd11walk_kernelILi3ELi4ELi1ELb0ELb0E|_ZN3fkd15overflow_kernel|_ZN3fkd17walk_round_kernel' \
    -c 6 -o gpurun_out/prof_bench $CMD > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
