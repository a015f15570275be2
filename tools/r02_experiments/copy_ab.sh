# host copy pool variants, one process each (FKD_COPY_THREADS / FKD_STREAM_COPY are read once per process)
for rep in 1 2; do
  for v in "FKD_STREAM_COPY=0" "FKD_STREAM_COPY=1" "FKD_STREAM_COPY=0;FKD_COPY_THREADS=16" "FKD_STREAM_COPY=1;FKD_COPY_THREADS=16" "FKD_STREAM_COPY=1;FKD_COPY_THREADS=12"; do
    env $(echo $v | tr ';' ' ') python tools/e2e_group_ab.py "" | sed "s/^default/$v/"
  done
done
