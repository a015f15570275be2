for lib in build/ab/lib_int.so paper_2210_12859_b200/libfkd_b200.so; do echo "lib $lib"
FKD_LIB=$PWD/$lib python tools/quickbench.py --configs fcp,knn4,knn8,knn16,knn32 --reps 3 2>&1 | grep true
FKD_LIB=$PWD/$lib python tools/quickbench.py --clustered --configs fcp,knn8 --reps 5 2>&1 | grep true
FKD_LIB=$PWD/$lib python tools/quickbench.py --dim 4 --m 2000000 --configs knn20,knn50,knn64 --reps 3 2>&1 | grep true
done
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
