python -m pytest tests -m gpu -x -q 2>&1 | tail -2
FKD_PERSIST=2 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for v in 0 2; do echo "persist $v"; FKD_PERSIST=$v python tools/quickbench.py --configs fcp,knn8 --reps 5 2>&1 | grep true; FKD_PERSIST=$v python tools/quickbench.py --clustered --configs fcp,knn8 --reps 5 2>&1 | grep true; done
