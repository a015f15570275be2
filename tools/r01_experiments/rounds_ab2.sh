# fcp round schedules with the final pass structure (first walk FKD_BUDGET,
# rounds FKD_RROUNDS_FCP, resume pass >= SMs x 64 survivors, CTA pass)
run() { echo "== $1 $2 $3"; env $2 python tools/quickbench.py $3 --configs $1 --reps 7 --sorted-only 2>&1 | grep cfg | cut -c1-100; }
for c in "--clustered" ""; do
  for v in "112 112,224,448" "112 112,224" "96 96,192" "112 112,336" "80 80,160,320" "128 128,384" "112 112,224,448,896" "144 144,288"; do set -- $v
    run fcp "FKD_BUDGET=$1 FKD_RROUNDS_FCP=$2" "$c"; done
done
