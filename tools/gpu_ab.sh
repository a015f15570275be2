python tools/quickbench.py --sorted-only --clustered --m 1250000 --configs fcp,knn8 --reps 5 2>&1 | grep true
python tools/quickbench.py --sorted-only --clustered --m 312500 --configs fcp,knn8 --reps 5 2>&1 | grep true
python tools/quickbench.py --sorted-only --clustered --configs fcp,knn8 --reps 3 2>&1 | grep true
python tools/quickbench.py --sorted-only --configs fcp,knn8 --reps 3 2>&1 | grep true
python tools/quickbench.py --sorted-only --dim 4 --m 2000000 --configs fcp,knn8 --reps 3 2>&1 | grep true
python tools/e2e_diag.py 2>&1 | grep auto
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
