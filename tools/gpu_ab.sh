python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/quickbench.py --sorted-only --clustered --configs fcp,knn8,knn16 --reps 2 2>&1 | grep true
python tools/quickbench.py --sorted-only --dim 4 --m 2000000 --configs knn50,knn64 --reps 2 2>&1 | grep true
python tools/quickbench.py --sorted-only --dim 8 --n 1000000 --m 200000 --configs fcp,knn8,knn16 --reps 2 2>&1 | grep true
