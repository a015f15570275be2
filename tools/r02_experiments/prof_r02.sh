# Round-2 profiling: launch list of the C3 bench step (concurrent submission),
# and one `ncu --set full` capture each of the C3 kNN8 first walk, the 4-D
# kNN50 walk and the 8-D kNN16 first walk.  usage: bash tools/prof_r02.sh <tag>
TAG=${1:-r02}
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pageable"
$B > gpurun_out/${TAG}_plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_ncu_launches.log 2>&1
echo "launch list exit $?"
K1="python tools/kernel_ab.py --dim 3 --k 8 --m 10000000 --clustered --reps 0"
$K1 > gpurun_out/${TAG}_plain_k1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 -o gpurun_out/${TAG}_knn8_walk $K1 > gpurun_out/${TAG}_ncu_k1.log 2>&1
echo "knn8 exit $?"
K2="python tools/kernel_ab.py --dim 4 --k 50 --m 1000000 --reps 0"
$K2 > gpurun_out/${TAG}_plain_k2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 -o gpurun_out/${TAG}_knn50_4d_walk $K2 > gpurun_out/${TAG}_ncu_k2.log 2>&1
echo "knn50 exit $?"
K3="python tools/kernel_ab.py --dim 8 --k 16 --m 200000 --reps 0"
$K3 > gpurun_out/${TAG}_plain_k3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 -o gpurun_out/${TAG}_knn16_8d_walk $K3 > gpurun_out/${TAG}_ncu_k3.log 2>&1
echo "knn16 8d exit $?"
ls -la gpurun_out/ | grep ${TAG}
