# 8-D kNN16 list in the output slot (product: FKD_SLOT_LIST_MIN_D=8, 4 blocks/SM) against the
# register list (build/ab/lib_noslot.so, -DFKD_SLOT_LIST_MIN_D=9), the slot list at 5 / 6 blocks/SM
# (lib_slot5 / lib_slot6: -DFKD_MINB_KB16_HIGH_D=5 / 6) and the slot list from 6-D up (lib_slotd6)
for lib in paper_2210_12859_b200/libfkd_b200.so build/ab/lib_noslot.so build/ab/lib_slot5.so build/ab/lib_slot6.so build/ab/lib_slotd6.so; do
  echo "== $lib"
  for d in 6 7 8; do
    FKD_LIB=$lib timeout 300 python tools/quickbench.py --dim $d --m 1000000 --configs knn16 --reps 3 --sorted-only 2>&1 | grep cfg | sed "s/^/d=$d /" | cut -c1-110
  done
done
