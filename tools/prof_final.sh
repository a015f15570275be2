# Final-code ncu evidence: launch list of the bench command, and `ncu --set full`
# of every walk-phase kernel of one C3 kNN8 batch and one C3 fcp batch
# (first walk, continuation rounds, resume pass, CTA pass).
# usage: bash tools/prof_final.sh <tag>
TAG=${1:-r02}
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pageable"
$B > gpurun_out/${TAG}_plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_ncu_launches.log 2>&1
echo "launch list exit $?"
for spec in "knn8:--dim 3 --k 8" "fcp:--dim 3 --k 1"; do
  name=${spec%%:*}; args=${spec#*:}
  K="python tools/kernel_ab.py $args --m 10000000 --clustered --reps 0"
  $K > gpurun_out/${TAG}_plain_$name.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k 'regex:walk_kernel|walk_round_kernel|overflow_kernel' -c 8 \
      -o gpurun_out/${TAG}_${name}_walk $K > gpurun_out/${TAG}_ncu_$name.log 2>&1
  echo "$name exit $?"
done
