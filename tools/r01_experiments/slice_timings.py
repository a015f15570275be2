"""Per-slice device timings (order / walk / tail ms) for slices of the C3 batch."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_12859_b200 as fk
m = 10_000_000
tree = fk.build_tree(fk.clustered_points(1, 1, m, 3))
dq = torch.from_numpy(fk.clustered_points(1, 2, m, 3)).cuda()
for kind, k in (("fcp", 1), ("knn", 8)):
    o = fk.BatchOptions(kind=fk.QueryKind[kind], k=k)
    for sl in (m, m // 8, m // 32):
        c = torch.empty(sl, dtype=torch.int32, device="cuda"); h = torch.empty(sl * k, dtype=torch.int64, device="cuda")
        for _ in range(3): _, t = fk.run_batch_device(tree, dq[:sl], c, h, o, timings=True)
        print(json.dumps({"kind": kind, "slice": sl, "timings": {a: b for a, b in t.items() if isinstance(b, (int, float))}}), flush=True)
