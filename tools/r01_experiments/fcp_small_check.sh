# product (rounds 112,224 below 2^22 queries) vs the previous schedule everywhere (FKD_RROUNDS_FCP=112,224,448)
for cfg in "--m 1000000 --n 1000000" "--clustered --m 1250000" "--clustered --m 2500000" "--dim 4 --m 1250000" "--dim 2 --m 1250000" "--clustered" "--dim 4"; do
  for s in "FKD_X=1" "FKD_RROUNDS_FCP=112,224,448"; do
    echo "== $cfg | $s"
    env $s timeout 300 python tools/quickbench.py $cfg --configs fcp --reps 5 --sorted-only 2>&1 | grep cfg | cut -c1-100
  done
done
