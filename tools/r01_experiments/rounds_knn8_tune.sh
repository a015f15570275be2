# kNN8 schedule re-tune after parked walks stopped writing their count (C3 clustered / uniform)
run() { echo "== $1 $2 $3"; env $2 python tools/quickbench.py $3 --configs $1 --reps 5 --sorted-only 2>&1 | grep cfg | sed 's/{"cfg": "[a-z0-9]*", "morton": true,//' | cut -c1-75; }
for c in "--clustered" ""; do
  run knn8 "FKD_BUDGET=-1" "$c"
  for v in "320 320,640,1280" "256 256,512,1024,2048" "448 448,896,1792" "512 512,1024,2048" "384 384,768,1536,3072"; do set -- $v
    run knn8 "FKD_BUDGET=$1 FKD_RROUNDS_KNN=$2" "$c"; done
done
