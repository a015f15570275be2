import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_12859_b200 as fk
for dim in (2, 3, 4):
    pts = fk.random_points(1, 1, 10_000_000, dim); tree = fk.build_tree(pts)
    qs = torch.from_numpy(fk.random_points(1, 2, 2_000_000, dim)).cuda()
    for k in ((8, 16, 20, 50) if dim != 3 else (8, 16)):
        c = torch.empty(len(qs), dtype=torch.int32, device="cuda"); h = torch.empty(len(qs) * k, dtype=torch.int64, device="cuda")
        o = fk.BatchOptions(kind=fk.QueryKind.knn, k=k)
        fk.run_batch_device(tree, qs, c, h, o)
        ts = [fk.run_batch_device(tree, qs, c, h, o, timings=True)[1]["walk_ms"] for _ in range(3)]
        print(json.dumps({"dim": dim, "k": k, "walk_ms": round(min(ts), 3)}), flush=True)
