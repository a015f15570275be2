for L in paper_2210_12859_b200/libfkd_b200.so paper_2210_12859_b200/libfkd_ab_m3.so paper_2210_12859_b200/libfkd_ab_m1.so; do
  FKD_LIB=$L python tools/kernel_ab.py --dim 5 --k 16 --m 2000000 --reps 2 | sed "s|^|$(basename $L) |; s/\"tail_ms\": [0-9.]*, //"
done
python tools/kernel_ab.py --dim 8 --k 16 --m 1000000 --reps 2 "" "FKD_BUDGET=1024" "FKD_BUDGET=8192" "FKD_RESUME_TRIPS=16384" "FKD_RESUME_TRIPS=-1" "FKD_BUDGET=100000" | sed "s/\"tail_ms\": [0-9.]*, //"
