# kNN walks (>= 8 slots): product (.cs on the Morton id, the query and the final stores) against
# .cs stores without .cs query loads (build/ab/lib_sq0.so: -DFKD_STREAM_QUERY_LOADS=0) and no .cs at all
# (build/ab/lib_nosio.so: -DFKD_STREAM_IO_MIN_KB=65); C3 clustered and uniform 3-D N = M = 10M, kNN8
for lib in paper_2210_12859_b200/libfkd_b200.so build/ab/lib_sq0.so build/ab/lib_nosio.so paper_2210_12859_b200/libfkd_b200.so build/ab/lib_sq0.so build/ab/lib_nosio.so; do
  echo "== $lib"
  FKD_LIB=$lib timeout 300 python tools/quickbench.py --clustered --configs knn8 --reps 5 --sorted-only 2>&1 | grep cfg | sed "s/^/clu /" | cut -c1-140
  FKD_LIB=$lib timeout 300 python tools/quickbench.py --configs knn8 --reps 5 --sorted-only 2>&1 | grep cfg | sed "s/^/uni /" | cut -c1-140
done
