# 3-D fcp walk body: explicit 8 steps (product) vs the unrolled loop (-DFKD_FCP_LOOP=1, build/ab/)
for rep in 1 2; do for lib in paper_2210_12859_b200/libfkd_b200.so build/ab/lib_fcploop.so; do
  echo "== $lib"
  for c in --clustered ""; do FKD_LIB=$lib python tools/quickbench.py $c --configs fcp --reps 5 --sorted-only 2>&1 | grep cfg | cut -c1-90; done
done; done
