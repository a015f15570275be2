# A/B of library builds on the C3 step (concurrent + serial) and single walks.
# usage: bash tools/lib_ab.sh <libA.so> <libB.so> [reps]
A=$1; B=$2; R=${3:-3}
for i in $(seq $R); do
  for L in $A $B; do
    echo "== $L"; FKD_LIB=$L python tools/step_ab.py concurrent serial --reps 1 --steps 10 | sed "s|^|$(basename $L) |"
  done
done
for L in $A $B; do
  for cfg in "--dim 3 --k 8 --m 10000000 --clustered" "--dim 3 --k 1 --m 10000000 --clustered" "--dim 4 --k 8 --m 4000000" "--dim 2 --k 16 --m 4000000" "--dim 4 --k 50 --m 1000000"; do
    FKD_LIB=$L python tools/kernel_ab.py $cfg | sed "s|^|$(basename $L) |"
  done
done
