# kNN16 in 5..8-D: product (4 blocks/SM for D >= 5) against build/ab/lib_hd1.so (-DFKD_MINB_KB16_HIGH_D=1)
for lib in paper_2210_12859_b200/libfkd_b200.so build/ab/lib_hd1.so; do
  echo "== $lib"
  for d in 5 6 7 8; do
    FKD_LIB=$lib timeout 300 python tools/quickbench.py --dim $d --m 1000000 --configs knn16 --reps 3 --sorted-only 2>&1 | grep cfg | sed "s/^/d=$d /" | cut -c1-110
  done
done
