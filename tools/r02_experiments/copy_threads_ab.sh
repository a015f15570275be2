for t in 8 12 16 8 12 16; do
  FKD_COPY_THREADS=$t python tools/pipe_trace.py --pageable 2>&1 | grep "^rep" | tr '\n' ' ' | sed "s/^/threads $t: /"; echo
done
