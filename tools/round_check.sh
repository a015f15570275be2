# Round-end style check on one B200: GPU tests, smoke, default bench, reference arm, launch list
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests exit $?"
tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench exit $?"; tail -c 3000 gpurun_out/bench_default.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref exit $?"; tail -c 1500 gpurun_out/bench_ref.json
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01j.csv $CMD > gpurun_out/ncu_launches_r01j.log 2>&1
python tools/launch_table.py gpurun_out/launches_r01j.csv "r01j launch list: bench.py --steps 2 --warmup 3 --no-cpu-baseline (C3)" > gpurun_out/r01j_bench_launches.md
head -14 gpurun_out/r01j_bench_launches.md
