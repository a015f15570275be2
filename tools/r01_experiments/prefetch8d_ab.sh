# (r01i: measured +5% with either variant; the FKD_PREFETCH experiment code was not kept)
# 8-D kNN16: prefetch of both children on a first visit (build/ab/lib_pf1.so: prefetch.global.L1,
# lib_pf2.so: prefetch.global.L2; -DFKD_PREFETCH=1/2) against the product
for lib in paper_2210_12859_b200/libfkd_b200.so build/ab/lib_pf1.so build/ab/lib_pf2.so paper_2210_12859_b200/libfkd_b200.so; do
  echo "== $lib"
  FKD_LIB=$lib timeout 300 python tools/quickbench.py --dim 8 --m 1000000 --configs knn16 --reps 3 --sorted-only 2>&1 | grep cfg | cut -c1-120
done
