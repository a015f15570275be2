# kNN16 walk occupancy: product (__launch_bounds__ min 1 block) against
# -DFKD_MINB_KB16=4 / 5 builds in build/ab/ (make EXTRA=-DFKD_MINB_KB16=v OUT=../../build/ab/lib_k16_v.so)
for lib in paper_2210_12859_b200/libfkd_b200.so build/ab/lib_k16_4.so build/ab/lib_k16_5.so; do
  echo "== $lib"
  FKD_LIB=$lib timeout 300 python tools/quickbench.py --dim 8 --m 1000000 --configs knn16 --reps 3 --sorted-only 2>&1 | grep cfg | cut -c1-110
  FKD_LIB=$lib timeout 300 python tools/quickbench.py --dim 4 --configs knn16 --reps 3 --sorted-only 2>&1 | grep cfg | cut -c1-110
  FKD_LIB=$lib timeout 300 python tools/quickbench.py --dim 2 --configs knn16 --reps 3 --sorted-only 2>&1 | grep cfg | cut -c1-110
  FKD_LIB=$lib timeout 300 python tools/quickbench.py --clustered --configs knn16 --reps 3 --sorted-only 2>&1 | grep cfg | cut -c1-110
done
