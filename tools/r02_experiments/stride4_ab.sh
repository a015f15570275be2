# 4-D store: 4 floats (plane selected by depth) vs 8 floats (plane in the padding, query rotated)
for L in build/ab/lib_s4.so build/ab/lib_s8.so build/ab/lib_s4.so build/ab/lib_s8.so; do
  for k in 1 4 8 16 50; do
    FKD_LIB=$L python tools/kernel_ab.py --dim 4 --k $k --m 4000000 --reps 2 | sed "s|^|$(basename $L) |" | cut -c1-120
  done
done
