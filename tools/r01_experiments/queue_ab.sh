# A/B of the work-queue walk (walk_queue_kernel, FKD_QUEUE=<first claim trips>,
# FKD_QUEUE_PARKS) against the default walk (+ rounds for fcp), C3 sizes
run() { echo "== $1 $2 $3"; env $2 python tools/quickbench.py $3 --configs $1 --reps 5 --sorted-only 2>&1 | grep cfg | cut -c1-120; }
for c in "--clustered" ""; do
  run knn8 "FKD_QUEUE=0" "$c"
  for v in "256 3" "128 3" "384 3" "192 3" "512 2"; do set -- $v; run knn8 "FKD_QUEUE=$1 FKD_QUEUE_PARKS=$2" "$c"; done
  run fcp "FKD_QUEUE=0" "$c"
  for v in "112 3" "64 3" "160 3"; do set -- $v; run fcp "FKD_QUEUE=$1 FKD_QUEUE_PARKS=$2" "$c"; done
done
