for b in 0 512 1024 2048 4096; do echo "budget $b"; FKD_BUDGET=$b python tools/quickbench.py --clustered --configs fcp,knn8 --reps 3 2>&1 | grep true; done
for b in 0 1024 4096; do echo "uniform budget $b"; FKD_BUDGET=$b python tools/quickbench.py --configs fcp,knn8 --reps 3 2>&1 | grep true; done
