# fcp distance: branch on first visit vs computed every trip (r01f: every trip won for 3-D, lost for 4-D;
# the product now computes it every trip for 3-D only). To rebuild the A/B, make the
# condition in LaneWalk::step a -D switch and build the variant into build/ab/lib_bf.so.
for lib in paper_2210_12859_b200/libfkd_b200.so build/ab/lib_bf.so; do
  echo "== $lib"
  for c in --clustered "" "--dim 4"; do
    FKD_LIB=$lib python tools/quickbench.py $c --configs fcp --reps 7 --sorted-only 2>&1 | grep cfg | cut -c1-100
  done
done
