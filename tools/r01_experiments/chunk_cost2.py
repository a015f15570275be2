"""Slices on concurrent streams: separates coherence loss from per-kernel tails."""
import json, os, sys, threading
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_12859_b200 as fk
m = 10_000_000
tree = fk.build_tree(fk.clustered_points(1, 1, m, 3))
dq = torch.from_numpy(fk.clustered_points(1, 2, m, 3)).cuda()
for kind, k in (("fcp", 1), ("knn", 8)):
    c = torch.empty(m, dtype=torch.int32, device="cuda"); h = torch.empty(m * k, dtype=torch.int64, device="cuda")
    o = fk.BatchOptions(kind=fk.QueryKind[kind], k=k)
    for parts in (1, 8):
        per = m // parts
        streams = [torch.cuda.Stream() for _ in range(parts)]
        def run(p):
            fk.run_batch_device(tree, dq[p*per:(p+1)*per], c[p*per:(p+1)*per], h[p*per*k:(p+1)*per*k], o, stream=streams[p])
        for rep in range(3):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for s in streams: s.wait_event(e0)
            ths = [threading.Thread(target=run, args=(p,)) for p in range(parts)]
            for t in ths: t.start()
            for t in ths: t.join()
            for s in streams: e1.wait(s) if False else None
            torch.cuda.synchronize(); e1.record(); e1.synchronize()
        print(json.dumps({"kind": kind, "parts": parts, "concurrent_ms": round(e0.elapsed_time(e1), 3)}), flush=True)
