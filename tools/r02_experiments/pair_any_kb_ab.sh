# packed-pair distance (FADD2/FMUL2) for 2-/3-D lists of more than 8 slots
for rep in 1 2; do
for L in build/ab/lib_p0.so build/ab/lib_p3.so; do
  for cfg in "--dim 2 --k 16 --m 4000000" "--dim 2 --k 20 --m 4000000" "--dim 3 --k 16 --m 4000000" "--dim 3 --k 50 --m 2000000" "--dim 2 --k 64 --m 2000000"; do
    FKD_LIB=$L python tools/kernel_ab.py $cfg --reps 2 | sed "s|^|$(basename $L) |" | cut -c1-120
  done
done
done
