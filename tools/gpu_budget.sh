python -m pytest tests/test_gpu_parity.py -x -q -k "overflow" 2>&1 | tail -3
for b in 0 1024 4096 16384; do echo "budget $b"; FKD_BUDGET=$b python tools/quickbench.py --clustered --configs fcp,knn8 --reps 3 2>&1 | grep true; done
FKD_BUDGET=4096 python tools/quickbench.py --configs fcp,knn8 --reps 3 2>&1 | grep true
