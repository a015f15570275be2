for o in morton tree; do echo "order $o"; export FKD_ORDER=$o
python tools/quickbench.py --sorted-only --configs fcp,knn8 --reps 3 2>&1 | grep true
python tools/quickbench.py --sorted-only --clustered --configs fcp,knn8 --reps 3 2>&1 | grep true
python tools/quickbench.py --sorted-only --dim 4 --m 2000000 --configs fcp,knn8 --reps 3 2>&1 | grep true
python tools/quickbench.py --sorted-only --dim 2 --configs fcp,knn16 --reps 3 2>&1 | grep true
done
FKD_ORDER=tree python -m pytest tests -m gpu -x -q -k "golden or hash or fuzz or dims" 2>&1 | tail -2
