# automatic walk block size (256 or 128 threads by resident warps) vs fixed 256
bash tools/lib_ab3.sh 1 build/ab/lib_base.so build/ab/lib_new.so
for L in build/ab/lib_base.so build/ab/lib_new.so; do
  for cfg in "--dim 4 --k 20 --m 2000000" "--dim 4 --k 32 --m 2000000" "--dim 4 --k 4 --m 4000000" "--dim 3 --k 16 --m 4000000" "--dim 3 --k 32 --m 2000000" "--dim 2 --k 50 --m 4000000" "--dim 5 --k 16 --m 1000000" "--dim 6 --k 8 --m 1000000" "--dim 4 --k 64 --m 1000000"; do
    FKD_LIB=$L python tools/kernel_ab.py $cfg --reps 2 | sed "s|^|$(basename $L) |; s/\"tail_ms\": [0-9.]*, //" | cut -c1-175
  done
done
