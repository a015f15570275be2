# (r01f) measured: every variant is slower than the default schedule; the 128-thread CTA
# variant of the overflow kernel it needs was not kept (FKD_OVF_T is not in the product).
# Tail passes: the last continuation rounds (latency-bound, few walks) against
# handing those walks to the CTA pass earlier, with 512- or 128-thread CTAs.
run() { echo "== $1 $2 $3"; env $2 python tools/quickbench.py $3 --configs $1 --reps 5 --sorted-only 2>&1 | grep cfg | sed 's/{"cfg": "[a-z0-9]*", "morton": true,//' | cut -c1-75; }
for c in "--clustered" ""; do
  run knn8 "FKD_OVF_T=512" "$c"
  run knn8 "FKD_OVF_T=128" "$c"
  run knn8 "FKD_RROUNDS_KNN=384,768 FKD_RESUME_MIN=1000000000000 FKD_BUDGET=384 FKD_OVF_T=128" "$c"
  run knn8 "FKD_RROUNDS_KNN=384,768 FKD_RESUME_MIN=1000000000000 FKD_BUDGET=384 FKD_OVF_T=512" "$c"
  run knn8 "FKD_RROUNDS_KNN=384 FKD_RESUME_MIN=1000000000000 FKD_BUDGET=384 FKD_OVF_T=128" "$c"
  run knn8 "FKD_RROUNDS_KNN=384,768 FKD_RESUME_MIN=1000000000000 FKD_BUDGET=384 FKD_OVF_T=128 FKD_OVF_CTAS=8" "$c"
  run fcp "FKD_OVF_T=512" "$c"
  run fcp "FKD_OVF_T=128" "$c"
  run fcp "FKD_RESUME_MIN=1000000000000 FKD_RROUNDS_FCP=112,224 FKD_OVF_T=128" "$c"
  run fcp "FKD_RESUME_MIN=1000000000000 FKD_RROUNDS_FCP=112,224 FKD_OVF_T=512" "$c"
  run fcp "FKD_RESUME_MIN=1000000000000 FKD_RROUNDS_FCP=112 FKD_OVF_T=128" "$c"
done
