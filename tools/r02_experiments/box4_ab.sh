# 4-D box pruning / 128-thread walk blocks, per list length (N = 10M uniform, M = 2M)
for L in build/ab/lib_base.so build/ab/lib_box4.so build/ab/lib_box4t128.so build/ab/lib_t128.so; do
  for k in 8 16 20 32 50; do
    FKD_LIB=$L python tools/kernel_ab.py --dim 4 --k $k --m 2000000 --reps 2 | sed "s|^|$(basename $L) |; s/\"tail_ms\": [0-9.]*, //" | cut -c1-175
  done
done
