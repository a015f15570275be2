# insertion network run from the list's end in blocks of 10, stopping at the first block no lane changes
for rep in 1 2; do
for L in build/ab/lib_cur.so build/ab/lib_tail.so; do
  for cfg in "--dim 4 --k 50 --m 2000000" "--dim 4 --k 20 --m 2000000" "--dim 3 --k 50 --m 2000000" "--dim 3 --k 20 --m 4000000" "--dim 2 --k 50 --m 4000000" "--dim 5 --k 20 --m 1000000"; do
    FKD_LIB=$L python tools/kernel_ab.py $cfg --reps 2 | sed "s|^|$(basename $L) |; s/\"tail_ms\": [0-9.]*, //" | cut -c1-150
  done
done
done
