# fcp schedule against batch size (device-resident walk ms incl. tail passes): default
# (budget 112, rounds 112,224,448) vs one budgeted walk + resume/CTA pass, vs shorter rounds
for cfg in "--m 1000000 --n 1000000" "--clustered --m 1250000" "--clustered --m 2500000" "--clustered --m 5000000" "--m 5000000"; do
  for s in "FKD_X=1" "FKD_BUDGET=448 FKD_RROUNDS_FCP=0" "FKD_BUDGET=1024 FKD_RROUNDS_FCP=0" "FKD_BUDGET=3072 FKD_RROUNDS_FCP=0" "FKD_RROUNDS_FCP=112,224"; do
    echo "== $cfg | $s"
    env $s timeout 300 python tools/quickbench.py $cfg --configs fcp --reps 5 --sorted-only 2>&1 | grep cfg | cut -c1-100
  done
done
