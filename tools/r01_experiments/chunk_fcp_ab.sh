# fcp walk schedule for chunk-sized batches (C3 clustered, 1.25M queries = one host-path chunk):
# device-resident quickbench per setting, then the host-path call (e2e_knobs) with the same settings
for s in "FKD_X=1" "FKD_RROUNDS_FCP=0" "FKD_BUDGET=448,FKD_RROUNDS_FCP=0" "FKD_BUDGET=1024,FKD_RROUNDS_FCP=0" "FKD_RROUNDS_FCP=112,224" "FKD_RROUNDS_FCP=224" "FKD_BUDGET=224,FKD_RROUNDS_FCP=224,448"; do
  echo "== $s"
  env $(echo $s | tr ',' ' ' | sed 's/FKD_RROUNDS_FCP=\([0-9]*\) \([0-9]\)/FKD_RROUNDS_FCP=\1,\2/') timeout 300 python tools/quickbench.py --clustered --m 1250000 --configs fcp --reps 5 --sorted-only 2>&1 | grep cfg | cut -c1-100
done
timeout 600 python tools/e2e_knobs.py "FKD_RROUNDS_FCP=0;FKD_X=1" "FKD_BUDGET=448;FKD_RROUNDS_FCP=0" "FKD_RROUNDS_FCP=112,224;FKD_X=1" "FKD_RROUNDS_FCP=224;FKD_X=1" "FKD_X=1"
