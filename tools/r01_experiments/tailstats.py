"""Per-query cost distribution of one workload on the GPU (development aid)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_12859_b200 as fk

dim = 3
for name, gen in (("clustered", lambda s, c: fk.clustered_points(1, s, c, dim)), ("uniform", lambda s, c: fk.random_points(1, s, c, dim))):
    pts = gen(1, 10_000_000); qs = gen(2, 10_000_000)
    tree = fk.KdTree.from_level_order(fk.build_level_order(pts))
    dq = torch.from_numpy(qs).cuda()
    for k in (1, 8):
        counts = torch.empty(len(qs), dtype=torch.int32, device="cuda")
        hits = torch.empty(len(qs) * k, dtype=torch.int64, device="cuda")
        pq = torch.empty(len(qs) * 3, dtype=torch.int64, device="cuda")
        opt = fk.BatchOptions(kind=fk.QueryKind.knn if k > 1 else fk.QueryKind.fcp, k=k, collect_stats=True)
        fk.run_batch_device(tree, dq, counts, hits, opt, per_query=pq)
        s = pq.view(-1, 3)[:, 0].cpu().numpy(); p = pq.view(-1, 3)[:, 2].cpu().numpy()
        top = np.argsort(s)[-3:]
        print(name, "k", k, "steps mean %.1f p99 %d p99.99 %d max %d | proc max %d" % (s.mean(), np.percentile(s, 99), np.percentile(s, 99.99), s.max(), p.max()), "top q", qs[top].tolist(), flush=True)
        _, tm = fk.run_batch_device(tree, dq, counts, hits, fk.BatchOptions(kind=opt.kind, k=k), timings=True)
        print("  walk_ms", tm["walk_ms"])
        # time the single slowest query alone
        one = dq[top[-1:]].contiguous()
        c1 = torch.empty(1, dtype=torch.int32, device="cuda"); h1 = torch.empty(k, dtype=torch.int64, device="cuda")
        fk.run_batch_device(tree, one, c1, h1, fk.BatchOptions(kind=opt.kind, k=k))
        _, tm = fk.run_batch_device(tree, one, c1, h1, fk.BatchOptions(kind=opt.kind, k=k), timings=True)
        print("  slowest query alone walk_ms", tm["walk_ms"], flush=True)
