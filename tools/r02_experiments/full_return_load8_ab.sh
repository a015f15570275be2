# 8-D (32-byte nodes, no plane slot): whole-node loads on return trips too
for rep in 1 2; do
for L in build/ab/lib_m4.so build/ab/lib_m8.so; do
  for cfg in "--k 16 --m 500000" "--k 8 --m 500000" "--k 1 --m 1000000" "--k 32 --m 200000"; do
    FKD_LIB=$L python tools/kernel_ab.py --dim 8 $cfg --reps 1 | sed "s|^|$(basename $L) |" | cut -c1-120
  done
done
done
