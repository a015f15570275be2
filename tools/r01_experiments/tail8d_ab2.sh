# resume-pass length (FKD_RESUME_TRIPS, trips) for 8-D kNN16 and the 4-D kNN16/64 configs that also use it
run() { echo "== $1 | $2"; env $1 timeout 300 python tools/quickbench.py $2 --reps 3 --sorted-only 2>&1 | grep cfg | sed 's/{"cfg": "\([a-z0-9]*\)", "morton": true,/\1/' | cut -c1-100; }
for t in 12288 24576 36864 49152 73728 98304; do run "FKD_RESUME_TRIPS=$t" "--dim 8 --m 1000000 --configs knn16"; done
run "FKD_RESUME_TRIPS=49152 FKD_BUDGET=6144" "--dim 8 --m 1000000 --configs knn16"
run "FKD_RESUME_TRIPS=49152 FKD_BUDGET=1536" "--dim 8 --m 1000000 --configs knn16"
for t in 12288 49152; do run "FKD_RESUME_TRIPS=$t" "--dim 4 --configs knn16,knn64,knn50"; done
for t in 12288 49152; do run "FKD_RESUME_TRIPS=$t" "--dim 5 --m 2000000 --configs knn16"; done
