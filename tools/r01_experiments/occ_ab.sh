# kNN8 walk occupancy: the product (44 registers, 5 blocks/SM) against a
# 6-blocks/SM build (-DFKD_MINB_KB8=6 -> 40 registers, 16 B of spills) in build/ab/
for lib in paper_2210_12859_b200/libfkd_b200.so build/ab/lib_mb6.so; do
  echo "== $lib"
  for c in --clustered "" "--dim 4"; do
    FKD_LIB=$lib python tools/quickbench.py $c --configs knn8 --reps 5 --sorted-only 2>&1 | grep cfg | cut -c1-100
  done
done
