# (r01i: Hilbert keys within ±1% everywhere, C3 kNN8 slightly slower; the FKD_HILBERT experiment code was not kept)
# Query order: Morton (product) vs Hilbert keys (build/ab/lib_hilbert.so, -DFKD_HILBERT=1), same 24-bit
# counting sort; walk + order ms
FKD_LIB=build/ab/lib_hilbert.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "uniform_all or tie_heavy or c1_c2" 2>&1 | tail -1
for rep in 1 2; do
for lib in paper_2210_12859_b200/libfkd_b200.so build/ab/lib_hilbert.so; do
  echo "== $lib"
  FKD_LIB=$lib timeout 300 python tools/quickbench.py --clustered --configs fcp,knn8 --reps 5 --sorted-only 2>&1 | grep cfg | cut -c1-100
  FKD_LIB=$lib timeout 300 python tools/quickbench.py --configs fcp,knn8 --reps 5 --sorted-only 2>&1 | grep cfg | cut -c1-100
  FKD_LIB=$lib timeout 300 python tools/quickbench.py --dim 4 --configs knn16 --reps 3 --sorted-only 2>&1 | grep cfg | cut -c1-100
  FKD_LIB=$lib timeout 300 python tools/quickbench.py --dim 2 --configs knn16 --reps 3 --sorted-only 2>&1 | grep cfg | cut -c1-100
done
done
