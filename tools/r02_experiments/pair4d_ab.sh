# packed-pair distance for 4-D lists of more than 8 slots
for rep in 1 2; do
for L in build/ab/lib_q3.so build/ab/lib_q4.so; do
  for k in 16 20 32 50; do
    FKD_LIB=$L python tools/kernel_ab.py --dim 4 --k $k --m 2000000 --reps 2 | sed "s|^|$(basename $L) |" | cut -c1-120
  done
done
done
