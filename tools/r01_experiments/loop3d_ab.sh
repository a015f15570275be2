# 3-D walks with the explicit body (product) vs the unrolled-loop body (-DFKD_LOOP_3D=1 build) for other k
# (r01h: build the variant by making the `W::kD == 3` test in walk_budgeted a -D switch)
for lib in paper_2210_12859_b200/libfkd_b200.so build/ab/lib_loop3d.so; do
  echo "== $lib"
  FKD_LIB=$lib python tools/quickbench.py --clustered --configs knn4,knn16,knn32,knn50 --reps 3 --sorted-only 2>&1 | grep cfg | cut -c1-90
done
