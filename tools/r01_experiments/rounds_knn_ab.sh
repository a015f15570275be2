# kNN8/16 continuation-round schedules with the final pass structure
run() { echo "== $1 $2 $3"; env $2 python tools/quickbench.py $3 --configs $1 --reps 5 --sorted-only 2>&1 | grep cfg | sed 's/{"cfg": "[a-z0-9]*", "morton": true,//' | cut -c1-75; }
for c in "--clustered" "" "--dim 4" "--dim 2"; do
  cfg=knn8; [ "$c" = "--dim 2" ] && cfg=knn16
  run $cfg "FKD_BUDGET=-1" "$c"
  for v in "256 256,512,1024,2048" "384 384,768,1536" "256 512,1024,2048" "512 512,1024,2048" "256 256,512,1024,2048,4096"; do set -- $v
    run $cfg "FKD_BUDGET=$1 FKD_RROUNDS_KNN=$2" "$c"; done
done
