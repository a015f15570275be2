# 9..16-D walk register caps (min blocks per SM 1 / 3 / 4 for 256-thread blocks)
for L in build/ab/lib_h1.so build/ab/lib_h3.so build/ab/lib_h4.so; do
  for cfg in "--dim 10 --k 8" "--dim 10 --k 1" "--dim 12 --k 8" "--dim 12 --k 16" "--dim 16 --k 8"; do
    FKD_LIB=$L python tools/kernel_ab.py $cfg --n 1000000 --m 200000 --reps 1 | sed "s|^|$(basename $L) |" | cut -c1-130
  done
done
