for L in build/ab/lib_m2.so build/ab/lib_m512.so build/ab/lib_m2048.so build/ab/lib_m2.so build/ab/lib_m512.so build/ab/lib_m2048.so; do
  echo "== $L"; FKD_LIB=$L python tools/latency.py 2>&1 | grep -v '"m": 100000'
done
