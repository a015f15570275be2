"""Host-path (fkd_run_batch) diagnosis: pinned copy bandwidth vs batch time."""
import ctypes as C, json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_12859_b200 as fk

def bw(nbytes, h2d):
    h = torch.empty(nbytes // 4, dtype=torch.float32).pin_memory()
    d = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")
    for _ in range(2):
        (d.copy_(h, non_blocking=True) if h2d else h.copy_(d, non_blocking=True)); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        (d.copy_(h, non_blocking=True) if h2d else h.copy_(d, non_blocking=True))
    torch.cuda.synchronize()
    return nbytes * 5 / (time.perf_counter() - t) / 1e9

print(json.dumps({"h2d_GBs": bw(1 << 30, True), "d2h_GBs": bw(1 << 30, False)}), flush=True)
m, dim = 10_000_000, 3
pts = fk.clustered_points(1, 1, m, dim)
tree = fk.build_tree(pts)
qs = fk.clustered_points(1, 2, m, dim)
hq = fk.LIB.fkd_host_alloc(qs.nbytes); C.memmove(hq, qs.ctypes.data, qs.nbytes)
for chunk in (None, 500_000, 1_000_000, 2_000_000, 4_000_000):
    if chunk: os.environ["FKD_CHUNK"] = str(chunk)
    else: os.environ.pop("FKD_CHUNK", None)
    rec = {"chunk": chunk or "auto"}
    for kind, k in (("fcp", 1), ("knn", 8)):
        hc = fk.LIB.fkd_host_alloc(m * 4); hh = fk.LIB.fkd_host_alloc(m * k * 8)
        o = fk.BatchOptions(kind=fk.QueryKind[kind], k=k).to_c()
        fk.LIB.fkd_run_batch(tree.handle, hq, m, dim, C.byref(o), hc, hh, None)
        ts = []
        for _ in range(3):
            t = time.perf_counter(); fk.LIB.fkd_run_batch(tree.handle, hq, m, dim, C.byref(o), hc, hh, None); ts.append(time.perf_counter() - t)
        rec[kind + "_ms"] = min(ts) * 1e3
        rec[kind + "_bytes_MB"] = (m * 12 + m * 4 + m * k * 8) / 1e6
        fk.LIB.fkd_host_free(hc); fk.LIB.fkd_host_free(hh)
    print(json.dumps(rec), flush=True)
