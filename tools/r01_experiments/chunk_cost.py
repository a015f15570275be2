"""Walk cost of sorting/walking a batch in slices (as the host pipeline does) vs whole."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_12859_b200 as fk
m = 10_000_000
tree = fk.build_tree(fk.clustered_points(1, 1, m, 3))
dq = torch.from_numpy(fk.clustered_points(1, 2, m, 3)).cuda()
for kind, k in (("fcp", 1), ("knn", 8)):
    c = torch.empty(m, dtype=torch.int32, device="cuda"); h = torch.empty(m * k, dtype=torch.int64, device="cuda")
    o = fk.BatchOptions(kind=fk.QueryKind[kind], k=k)
    for parts in (1, 4, 8, 16):
        per = m // parts
        tot = 0.0
        for rep in range(2):
            t = 0.0
            for p in range(parts):
                _, tm = fk.run_batch_device(tree, dq[p*per:(p+1)*per], c[p*per:(p+1)*per], h[p*per*k:(p+1)*per*k], o, timings=True)
                t += tm["walk_ms"] + tm["order_ms"]
            tot = t
        print(json.dumps({"kind": kind, "parts": parts, "ms": round(tot, 3)}), flush=True)
