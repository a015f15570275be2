# A/B of the store-layout experiments (profiles/r01e_ab_store_layout.log):
# top levels of the tree in shared memory (FKD_SMEM_LEVELS=L) and a
# structure-of-arrays 3-D store (FKD_SOA=1).  Both lost and are not in the
# product; to rebuild the variants:
#   git apply tools/experiments/store_layout_smem_soa.patch
#   cd paper_2210_12859_b200/csrc
#   for L in 0 8 10 11; do make EXTRA=-DFKD_SMEM_LEVELS=$L OBJDIR=/tmp/ab/obj_s$L OUT=../../build/ab/lib_s$L.so; done
#   make EXTRA=-DFKD_SOA=1 OBJDIR=/tmp/ab/obj_soa OUT=../../build/ab/lib_soa.so
#   git apply -R ../../tools/experiments/store_layout_smem_soa.patch
# (the SoA variant only converts the register-list walk and the tail passes;
# the heap / trace kernels still read row-major, hence its parity failure.)
for v in s0 s8 s10 s11 soa; do
  echo "== $v"
  FKD_LIB=build/ab/lib_$v.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "uniform_all or tie_heavy or overflow or c1_c2 or degenerate" 2>&1 | tail -1
  for c in "" "--clustered"; do
    FKD_LIB=build/ab/lib_$v.so timeout 300 python tools/quickbench.py $c --configs fcp,knn8 --reps 5 --sorted-only 2>&1 | grep cfg
  done
done
