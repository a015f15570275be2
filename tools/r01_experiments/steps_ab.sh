# kNN steps per budget check: explicit 4-step body (lib_old, HEAD) vs the unrolled-loop
# body with 4 / 2 / 8 steps (-DFKD_KNN_STEPS=n builds in build/ab/)
for rep in 1 2; do
for lib in build/ab/lib_old.so paper_2210_12859_b200/libfkd_b200.so build/ab/lib_steps2.so build/ab/lib_steps8.so; do
  echo "== $lib"
  for c in --clustered "" "--dim 4"; do
    FKD_LIB=$lib python tools/quickbench.py $c --configs knn8 --reps 5 --sorted-only 2>&1 | grep cfg | cut -c1-100
  done
done
done
