"""Host-path (fkd_run_batch, pinned buffers) time under pipeline knobs, C3 (development aid).
Usage: python tools/e2e_knobs.py 'FKD_FIRST_BUDGET_DIV=4,FKD_CHUNK_DIV=16' ..."""
import ctypes as C, json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_12859_b200 as fk

m, dim = 10_000_000, 3
tree = fk.build_tree(fk.clustered_points(1, 1, m, dim))
qs = fk.clustered_points(1, 2, m, dim)
hq = fk.LIB.fkd_host_alloc(qs.nbytes); C.memmove(hq, qs.ctypes.data, qs.nbytes)
bufs = {k: (fk.LIB.fkd_host_alloc(m * 4), fk.LIB.fkd_host_alloc(m * k * 8)) for k in (1, 8)}
base = dict(os.environ)
for spec in [""] + sys.argv[1:]:
    env = dict(kv.split("=", 1) for kv in spec.split(";" if ";" in spec else ",") if kv)  # ";" separates knobs whose values hold commas
    os.environ.clear(); os.environ.update(base); os.environ.update(env)
    rec = {"knobs": spec or "default"}
    for kind, k in (("fcp", 1), ("knn", 8)):
        o = fk.BatchOptions(kind=fk.QueryKind[kind], k=k).to_c()
        hc, hh = bufs[k]
        ts = []
        for rep in range(6):
            t = time.perf_counter()
            rc = fk.LIB.fkd_run_batch(tree.handle, hq, m, dim, C.byref(o), hc, hh, None)
            ts.append(time.perf_counter() - t)
            assert rc == 0
        rec[kind + "_ms"] = round(float(np.median(ts[1:])) * 1e3, 2)
        rec[kind + "_min"] = round(min(ts[1:]) * 1e3, 2)
    rec["e2e_Gqps"] = round(2 * m / (rec["fcp_ms"] + rec["knn_ms"]) / 1e6, 3)
    print(json.dumps(rec), flush=True)
