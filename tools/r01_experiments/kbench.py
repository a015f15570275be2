"""Large-k timing on the paper's 4-D setting (N=10M, M=2M): register buckets vs the heap kernel."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_12859_b200 as fk
pts = fk.random_points(1, 1, 10_000_000, 4)
tree = fk.build_tree(pts)
qs = torch.from_numpy(fk.random_points(1, 2, 2_000_000, 4)).cuda()
for k in (16, 20, 32, 50, 64):
    for r in (float("inf"), 0.01):
        c = torch.empty(len(qs), dtype=torch.int32, device="cuda"); h = torch.empty(len(qs) * k, dtype=torch.int64, device="cuda")
        o = fk.BatchOptions(kind=fk.QueryKind.knn, k=k, max_radius=r)
        fk.run_batch_device(tree, qs, c, h, o)
        ts = [fk.run_batch_device(tree, qs, c, h, o, timings=True)[1]["walk_ms"] for _ in range(2)]
        print(json.dumps({"k": k, "r": r, "heap": os.environ.get("FKD_REG_MAXK", "64"), "walk_ms": min(ts)}), flush=True)
