bash tools/lib_ab3.sh 2 build/ab/lib_base.so build/ab/lib_pred.so
for L in build/ab/lib_base.so build/ab/lib_pred.so; do
  for cfg in "--dim 3 --k 16 --m 4000000" "--dim 4 --k 16 --m 2000000" "--dim 3 --k 4 --m 4000000"; do
    FKD_LIB=$L python tools/kernel_ab.py $cfg | sed "s|^|$(basename $L) |; s/\"tail_ms\": [0-9.]*, //" | cut -c1-170
  done
done
