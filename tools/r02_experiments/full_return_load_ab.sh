# 4-D (16-byte nodes, no plane slot): a return trip loads the whole node (one vector, same sector) vs the split coordinate only
for rep in 1 2; do
for L in build/ab/lib_r0.so build/ab/lib_r1.so; do
  for k in 1 4 8 16 20 50; do
    FKD_LIB=$L python tools/kernel_ab.py --dim 4 --k $k --m 4000000 --reps 2 | sed "s|^|$(basename $L) |" | cut -c1-120
  done
  FKD_LIB=$L python tools/kernel_ab.py --dim 4 --k 16 --m 2000000 --clustered --reps 2 | sed "s|^|$(basename $L) clustered |" | cut -c1-130
done
done
