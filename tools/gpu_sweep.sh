python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for p in 0 1; do FKD_PERSIST=$p python tools/quickbench.py --configs fcp,knn8 --reps 3 2>&1 | grep true; done
for r in 1 4 16; do echo refill $r; FKD_REFILL=$r python tools/quickbench.py --configs fcp,knn8 --reps 3 2>&1 | grep true; done
for p in 0 1; do FKD_PERSIST=$p python tools/quickbench.py --clustered --configs fcp,knn8 --reps 3 2>&1 | grep cfg; done
