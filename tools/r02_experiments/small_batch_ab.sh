for L in build/ab/lib_nosmall.so build/ab/lib_small.so build/ab/lib_nosmall.so build/ab/lib_small.so; do
  echo "== $L"; FKD_LIB=$L python tools/latency.py 2>&1 | grep -v '"m": 100000'
done
