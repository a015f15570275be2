echo "quickbench default"; python tools/quickbench.py --clustered --configs fcp,knn8 --reps 5 --sorted-only 2>&1 | grep cfg | cut -c1-110
echo "quickbench old"; FKD_RROUNDS_KNN=0 FKD_BUDGET=3072 python tools/quickbench.py --clustered --configs knn8 --reps 5 --sorted-only 2>&1 | grep cfg | cut -c1-110
echo "matrix default"; python tools/matrix.py --only c3 2>/dev/null | cut -c1-330
echo "matrix old knn"; FKD_RROUNDS_KNN=0 FKD_BUDGET_ORDERED=3072 python tools/matrix.py --only c3 2>/dev/null | cut -c1-330
