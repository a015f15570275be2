# Round-end style check on one B200: GPU tests, smoke, default bench, reference arm.
# usage (from gpurun): bash tools/round_check.sh <tag>
TAG=${1:-r02}
set -x
timeout 1800 python -m pytest tests -m gpu -x -q -rs > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "gpu tests exit $?"
tail -5 gpurun_out/${TAG}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --steps 10 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench exit $?"; tail -c 4000 gpurun_out/${TAG}_bench.json; tail -5 gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; echo "ref exit $?"; tail -c 2000 gpurun_out/${TAG}_bench_ref.json
