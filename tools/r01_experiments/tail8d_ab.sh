# 8-D kNN16 (C4, N=10M, M=1M): first-walk budget and resume-pass length against the CTA pass
run() { echo "== $1"; env $1 timeout 300 python tools/quickbench.py --dim 8 --m 1000000 --configs knn16 --reps 3 --sorted-only 2>&1 | grep cfg | sed 's/{"cfg": "[a-z0-9]*", "morton": true,//' | cut -c1-110; }
run "FKD_X=default"
run "FKD_RESUME_TRIPS=-1"
run "FKD_RESUME_TRIPS=49152"
run "FKD_BUDGET=0"
run "FKD_BUDGET=12288"
run "FKD_BUDGET=12288 FKD_RESUME_TRIPS=-1"
run "FKD_RESUME_MIN=1000000000000"
