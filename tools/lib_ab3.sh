# A/B/C of library builds: C3 step (concurrent + serial) x reps, then single walks.
# usage: bash tools/lib_ab3.sh <reps> <lib> <lib> [<lib> ...]
R=$1; shift
for i in $(seq $R); do
  for L in "$@"; do
    FKD_LIB=$L python tools/step_ab.py concurrent serial --reps 1 --steps 10 | sed "s|^|$(basename $L) |"
  done
done
for L in "$@"; do
  for cfg in "--dim 3 --k 8 --m 10000000 --clustered" "--dim 3 --k 1 --m 10000000 --clustered" "--dim 4 --k 8 --m 4000000" "--dim 2 --k 16 --m 4000000" "--dim 4 --k 50 --m 1000000" "--dim 8 --k 16 --m 500000"; do
    FKD_LIB=$L python tools/kernel_ab.py $cfg | sed "s|^|$(basename $L) |; s/\"tail_ms\": [0-9.]*, //" | cut -c1-150
  done
done
