for b in 768 1024 1536; do echo "fcp budget $b"; FKD_BUDGET=$b python tools/quickbench.py --clustered --configs fcp --reps 5 2>&1 | grep true; done
for b in 2048 3072 4096; do echo "knn budget $b"; FKD_BUDGET=$b python tools/quickbench.py --clustered --configs knn8 --reps 5 2>&1 | grep true; done
