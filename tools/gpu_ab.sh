python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in 0; do FKD_WAVE=$v python tools/quickbench.py --configs fcp,knn8 --reps 3 2>&1 | grep true; FKD_WAVE=$v python tools/quickbench.py --clustered --configs fcp,knn8 --reps 3 2>&1 | grep true; done
python bench.py --steps 10 > gpurun_out/bench_e2e.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bench_e2e.json')); print(d['value']/1e6, d['e2e'], d['per_batch'])"
