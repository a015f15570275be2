for L in paper_2210_12859_b200/libfkd_ab_nobox.so paper_2210_12859_b200/libfkd_b200.so; do
  for cfg in "--dim 4 --k 8 --m 4000000" "--dim 4 --k 50 --m 2000000" "--dim 4 --k 1 --m 4000000" "--dim 4 --k 16 --m 4000000" "--dim 5 --k 16 --m 1000000" "--dim 6 --k 8 --m 1000000" "--dim 8 --k 16 --m 1000000"; do
    FKD_LIB=$L python tools/kernel_ab.py $cfg --reps 2 | sed "s|^|$(basename $L) |; s/\"tail_ms\": [0-9.]*, //"
  done
done
