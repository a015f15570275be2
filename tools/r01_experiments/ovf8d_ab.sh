# 8-D kNN16 CTA pass: 512-thread CTAs (product) vs 256 (build/ab/lib_ovf256.so: the r01i experiment
# built launch_overflow with T = 256 for D == 8), CTAs per SM (measured: within 1%, not kept)
run() { echo "== $1 $2"; env $2 FKD_LIB=$1 timeout 300 python tools/quickbench.py --dim 8 --m 1000000 --configs knn16 --reps 3 --sorted-only 2>&1 | grep cfg | cut -c1-120; }
for c in 1 2 4 8; do
  run paper_2210_12859_b200/libfkd_b200.so FKD_OVF_CTAS=$c
  run build/ab/lib_ovf256.so FKD_OVF_CTAS=$c
done
