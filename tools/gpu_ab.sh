FKD_QPL=8 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
echo base; python tools/quickbench.py --configs fcp,knn8 --reps 3 2>&1 | grep true; python tools/quickbench.py --clustered --configs fcp,knn8 --reps 3 2>&1 | grep true
for q in 4 8 16; do for r in 4 8 16; do echo "qpl $q refill $r"; FKD_QPL=$q FKD_REFILL=$r python tools/quickbench.py --configs fcp --reps 3 2>&1 | grep true; done; done
