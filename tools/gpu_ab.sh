python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for v in 0 1; do echo "align $v"; FKD_SIBLING_ALIGN=$v python tools/quickbench.py --configs fcp,knn8 --reps 5 2>&1 | grep true; FKD_SIBLING_ALIGN=$v python tools/quickbench.py --clustered --configs fcp,knn8 --reps 5 2>&1 | grep true; done
