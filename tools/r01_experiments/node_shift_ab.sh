# Tree store shifted by one slot (FKD_NODE_SHIFT=1: siblings 2c+1 / 2c+2 share a 32-byte sector for
# 16-byte nodes) against the unshifted store; walk ms, N = 10M
for sh in 0 1 0 1; do
  echo "== shift $sh"
  export FKD_NODE_SHIFT=$sh
  timeout 300 python tools/quickbench.py --clustered --configs fcp,knn8 --reps 5 --sorted-only 2>&1 | grep cfg | sed "s/^/3d-clu /" | cut -c1-110
  timeout 300 python tools/quickbench.py --configs fcp,knn8 --reps 5 --sorted-only 2>&1 | grep cfg | sed "s/^/3d-uni /" | cut -c1-110
  timeout 300 python tools/quickbench.py --dim 4 --m 2000000 --configs knn16 --reps 3 --sorted-only 2>&1 | grep cfg | sed "s/^/4d /" | cut -c1-110
  timeout 300 python tools/quickbench.py --dim 2 --m 2000000 --configs knn16 --reps 3 --sorted-only 2>&1 | grep cfg | sed "s/^/2d /" | cut -c1-110
done
