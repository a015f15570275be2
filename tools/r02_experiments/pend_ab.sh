for L in build/ab/lib_base.so build/ab/lib_p2.so build/ab/lib_p3.so build/ab/lib_p4.so; do
  for cfg in "--dim 4 --k 20 --m 2000000" "--dim 4 --k 32 --m 2000000" "--dim 4 --k 50 --m 2000000" "--dim 4 --k 64 --m 1000000" "--dim 3 --k 50 --m 2000000" "--dim 2 --k 20 --m 4000000" "--dim 6 --k 20 --m 200000"; do
    FKD_LIB=$L timeout 300 python tools/kernel_ab.py $cfg --reps 3 | sed "s|^|$(basename $L) |; s/\"tail_ms\": [0-9.]*, //"
  done
done
