# kNN distance on a first visit only (build/ab/lib_kdb.so: -DFKD_KNN_DIST_BRANCH=1) against the
# product (distance every trip, admission predicated); walk ms, N = 10M
for lib in paper_2210_12859_b200/libfkd_b200.so build/ab/lib_kdb.so paper_2210_12859_b200/libfkd_b200.so build/ab/lib_kdb.so; do
  echo "== $lib"
  FKD_LIB=$lib timeout 300 python tools/quickbench.py --clustered --configs knn8 --reps 5 --sorted-only 2>&1 | grep cfg | sed "s/^/3d-clu /" | cut -c1-110
  FKD_LIB=$lib timeout 300 python tools/quickbench.py --configs knn8 --reps 5 --sorted-only 2>&1 | grep cfg | sed "s/^/3d-uni /" | cut -c1-110
  FKD_LIB=$lib timeout 300 python tools/quickbench.py --dim 4 --m 2000000 --configs knn8,knn16 --reps 3 --sorted-only 2>&1 | grep cfg | sed "s/^/4d /" | cut -c1-110
  FKD_LIB=$lib timeout 300 python tools/quickbench.py --dim 2 --m 2000000 --configs knn16 --reps 3 --sorted-only 2>&1 | grep cfg | sed "s/^/2d /" | cut -c1-110
  FKD_LIB=$lib timeout 300 python tools/quickbench.py --dim 8 --m 200000 --configs knn16 --reps 2 --sorted-only 2>&1 | grep cfg | sed "s/^/8d /" | cut -c1-110
done
