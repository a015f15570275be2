for i in 1 2; do for L in paper_2210_12859_b200/libfkd_b200.so paper_2210_12859_b200/libfkd_ab_cells0.5.so paper_2210_12859_b200/libfkd_ab_cells0.2.so; do
  FKD_LIB=$L python tools/step_ab.py concurrent --reps 1 --steps 10 | sed "s|^|$(basename $L) |"
done; done
for L in paper_2210_12859_b200/libfkd_b200.so paper_2210_12859_b200/libfkd_ab_cells0.5.so paper_2210_12859_b200/libfkd_ab_cells0.2.so; do
  FKD_LIB=$L python tools/step_timeline.py | tail -1 | sed "s|^|$(basename $L) |"
done
