# Preferred shared-memory carveout of the walk kernels (FKD_L1_CARVEOUT percent; unset = driver's choice)
for c in unset 0 unset 0 50; do
  echo "== carveout $c"
  if [ $c = unset ]; then unset FKD_L1_CARVEOUT; else export FKD_L1_CARVEOUT=$c; fi
  timeout 300 python tools/quickbench.py --clustered --configs fcp,knn8 --reps 5 --sorted-only 2>&1 | grep cfg | sed "s/^/clu /" | cut -c1-110
  timeout 300 python tools/quickbench.py --configs knn8 --reps 5 --sorted-only 2>&1 | grep cfg | sed "s/^/uni /" | cut -c1-110
done
