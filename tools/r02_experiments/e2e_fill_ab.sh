# host fill of unbounded-radius counts vs DMA, copy-pool width / stores (one process per variant)
for rep in 1 2; do
for v in "X=0" "FKD_HOST_COUNTS=0" "FKD_COPY_THREADS=4" "FKD_STREAM_COPY=0" "FKD_COPY_THREADS=2;FKD_STREAM_COPY=0"; do
  env $(echo $v | tr ';' ' ') python tools/e2e_pipelined_ab.py "" | sed "s/^default/$v/"
done
done
