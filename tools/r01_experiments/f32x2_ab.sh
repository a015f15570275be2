# A/B of the packed-pair squared distance (FADD2/FMUL2): the product library against one
# built with pairs off.  Build the reference variant with an FKD_F32X2 switch in sq_dist
# (the r01f experiment used -DFKD_F32X2_MAX_D=0 on the then-current source) into build/ab/lib_nof2.so.
for lib in paper_2210_12859_b200/libfkd_b200.so build/ab/lib_nof2.so; do
  echo "== $lib"
  FKD_LIB=$lib python tools/quickbench.py --dim 4 --configs knn20,knn8 --reps 3 --sorted-only 2>&1 | grep cfg | cut -c1-110
  FKD_LIB=$lib FKD_RESUME_MIN=1000000000 python tools/quickbench.py --dim 4 --configs knn20 --reps 3 --sorted-only 2>&1 | grep cfg | cut -c1-110
  FKD_LIB=$lib python tools/quickbench.py --dim 8 --m 1000000 --configs knn16 --reps 2 --sorted-only 2>&1 | grep cfg | cut -c1-110
  FKD_LIB=$lib python tools/quickbench.py --clustered --configs fcp,knn8 --reps 5 --sorted-only 2>&1 | grep cfg | cut -c1-110
  FKD_LIB=$lib python tools/quickbench.py --n 1000000 --m 1000000 --configs knn8,knn8r01 --reps 5 --sorted-only 2>&1 | grep cfg | cut -c1-110
  FKD_LIB=$lib FKD_RROUNDS_KNN=0 FKD_BUDGET=3072 python tools/quickbench.py --n 1000000 --m 1000000 --configs knn8,knn8r01 --reps 5 --sorted-only 2>&1 | grep cfg | cut -c1-110
done
