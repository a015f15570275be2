# fcp keys with the walk's 1-based node id vs the 0-based one
for rep in 1 2; do
for L in build/ab/lib_n0.so build/ab/lib_n1.so; do
  FKD_LIB=$L python tools/step_ab.py concurrent --reps 1 --steps 10 | sed "s|^|$(basename $L) |"
  for cfg in "--dim 3 --k 1 --m 10000000 --clustered" "--dim 3 --k 1 --m 10000000" "--dim 2 --k 1 --m 4000000" "--dim 4 --k 1 --m 4000000" "--dim 6 --k 1 --m 1000000" "--dim 10 --k 1 --n 1000000 --m 200000"; do
    FKD_LIB=$L python tools/kernel_ab.py $cfg --reps 2 | sed "s|^|$(basename $L) |" | cut -c1-110
  done
done
done
