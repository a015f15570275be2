FKD_QPL=4 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for v in 1 2 4 8; do echo "qpl $v"; FKD_QPL=$v python tools/quickbench.py --configs fcp,knn8 --reps 3 2>&1 | grep true; FKD_QPL=$v python tools/quickbench.py --clustered --configs fcp,knn8 --reps 3 2>&1 | grep true; done
