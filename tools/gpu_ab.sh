python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do python tools/quickbench.py --configs fcp,knn8 --reps 5 2>&1 | grep true; python tools/quickbench.py --clustered --configs fcp,knn8 --reps 5 2>&1 | grep true; done
