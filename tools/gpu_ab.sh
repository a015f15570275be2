for lib in build/ab/lib_bub.so paper_2210_12859_b200/libfkd_b200.so build/ab/lib_s8.so; do echo "lib $lib"; FKD_LIB=$PWD/$lib python tools/kbench2.py; done
