# 2-D store: packed 8-byte nodes vs 16-byte nodes with the split plane in the padding
# (r01h: run when the latter was FKD_LAYOUT=padded2d; it is now the default and
# FKD_LAYOUT=packed selects the 8-byte store), C4-2D sizes
FKD_LAYOUT=padded2d timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "uniform_all or tie_heavy or overflow or degenerate" 2>&1 | tail -1
for rep in 1 2; do for lay in packed2 padded2d; do
  echo "== $lay"; FKD_LAYOUT=$lay python tools/quickbench.py --dim 2 --configs knn16,fcp,knn8 --reps 5 --sorted-only 2>&1 | grep cfg | cut -c1-90
done; done
