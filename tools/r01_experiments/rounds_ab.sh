# A/B of the continuation rounds (walk_round_kernel) on C3-sized batches:
# first-walk budget FKD_BUDGET, then FKD_RROUNDS_{FCP,KNN} trips per round.
run() { echo "== $1 $2 $3 $4"; env $2 python tools/quickbench.py $3 --configs $1 --reps 5 --sorted-only 2>&1 | grep cfg | cut -c1-140; }
for c in "--clustered" ""; do
  run fcp "FKD_BUDGET=-1" "$c"
  for v in "128 128,256" "96 96,192,384" "128 128,128,256" "160 160,320" "112 112,224,448" "128 128,256,512,1024"; do set -- $v
    run fcp "FKD_BUDGET=$1 FKD_RROUNDS_FCP=$2" "$c"; done
  run knn8 "FKD_BUDGET=-1" "$c"
  for v in "256 256,512" "320 320,640" "192 192,384,768" "256 256,256,512" "384 384,768" "256 256,512,1024,2048"; do set -- $v
    run knn8 "FKD_BUDGET=$1 FKD_RROUNDS_KNN=$2" "$c"; done
done
