# fcp rounds 112,224,448 (default) vs 112,224 at C3 size (10M clustered / uniform), 3 alternations
for rep in 1 2 3; do
  for s in "FKD_X=1" "FKD_RROUNDS_FCP=112,224"; do
    echo "== $s"
    env $s timeout 300 python tools/quickbench.py --clustered --configs fcp --reps 7 --sorted-only 2>&1 | grep cfg | cut -c1-100
    env $s timeout 300 python tools/quickbench.py --configs fcp --reps 7 --sorted-only 2>&1 | grep cfg | cut -c1-100
  done
done
