python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/quickbench.py --configs fcp,knn8 --reps 3 2>&1 | grep true; python tools/quickbench.py --clustered --configs fcp,knn8 --reps 3 2>&1 | grep true
for b in 8 7 6; do echo "mbits $b"; FKD_MORTON_BITS=$b python tools/quickbench.py --configs fcp,knn8 --reps 3 2>&1 | grep true; FKD_MORTON_BITS=$b python tools/quickbench.py --clustered --configs fcp,knn8 --reps 3 2>&1 | grep true; done
