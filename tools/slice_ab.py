import sys, os, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2210_12859_b200 as fk
dev = torch.device("cuda", 0)
n = m = 10_000_000
nodes = fk.build_level_order_device(torch.from_numpy(fk.clustered_points(1, 1, n, 3)).to(dev))
tree = fk.KdTree.from_device(nodes)
q = torch.from_numpy(fk.clustered_points(1, 2, m, 3)).to(dev)
for kind, k in ((fk.QueryKind.knn, 8), (fk.QueryKind.fcp, 1)):
    for parts in (1, 2, 4, 8, 16):
        per = m // parts
        c = torch.empty(per, dtype=torch.int32, device=dev); h = torch.empty(per * k, dtype=torch.int64, device=dev)
        tot = []
        for rep in range(3):
            s = 0.0
            for p in range(parts):
                qq = q[p * per:(p + 1) * per]
                _, tm = fk.run_batch_device(tree, qq, c, h, fk.BatchOptions(kind=kind, k=k), timings=True)
                s += tm["order_ms"] + tm["walk_ms"]
            tot.append(s)
        print(kind.name, k, "parts", parts, "sum ms %.3f" % np.median(tot), flush=True)
