# packed-pair distance for 5..16-D lists of up to 16 slots
for rep in 1 2; do
for L in build/ab/lib_h0.so build/ab/lib_h1.so; do
  for cfg in "--dim 5 --k 16 --m 1000000" "--dim 5 --k 1 --m 2000000" "--dim 6 --k 8 --m 1000000" "--dim 8 --k 16 --m 500000" "--dim 8 --k 8 --m 500000" "--dim 8 --k 1 --m 1000000" "--dim 10 --k 8 --n 1000000 --m 200000"; do
    FKD_LIB=$L python tools/kernel_ab.py $cfg --reps 1 | sed "s|^|$(basename $L) |" | cut -c1-120
  done
done
done
