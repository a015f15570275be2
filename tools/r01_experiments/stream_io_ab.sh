# Evict-first (.cs) query loads and result stores for every list size (build/ab/lib_sio.so: -DFKD_STREAM_IO_MIN_KB=1) against
# the code without them (-DFKD_STREAM_IO_MIN_KB=65, the product before r01j; the product now uses them from 8 slots up),
# C3 clustered and uniform 3-D N = M = 10M, fcp + kNN8
for lib in paper_2210_12859_b200/libfkd_b200.so build/ab/lib_sio.so paper_2210_12859_b200/libfkd_b200.so build/ab/lib_sio.so; do
  echo "== $lib"
  FKD_LIB=$lib timeout 300 python tools/quickbench.py --clustered --configs fcp,knn8 --reps 5 --sorted-only 2>&1 | grep cfg | sed "s/^/clu /" | cut -c1-140
  FKD_LIB=$lib timeout 300 python tools/quickbench.py --configs fcp,knn8 --reps 5 --sorted-only 2>&1 | grep cfg | sed "s/^/uni /" | cut -c1-140
done
for lib in paper_2210_12859_b200/libfkd_b200.so build/ab/lib_sio.so; do
  FKD_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench $lib', round(d['value']/1e6,1), {k: round(v['walk_ms'],3) for k,v in d['per_batch'].items()}, round(d['e2e']['value']/1e6,1))"
done
