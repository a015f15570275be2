for c in "" "--clustered"; do
  echo "== base $c"; python tools/quickbench.py $c --configs fcp,knn8 --reps 5 --sorted-only 2>&1 | grep cfg | cut -c1-120
  for r in "64,64,128,256,512,1024" "128,128,256,512,1024" "160,160,320,320,640,1024" "256,512,1024"; do
    echo "== wave $r $c"; FKD_WAVE=1 FKD_ROUNDS=$r python tools/quickbench.py $c --configs fcp,knn8 --reps 5 --sorted-only 2>&1 | grep cfg | cut -c1-120
  done
done
