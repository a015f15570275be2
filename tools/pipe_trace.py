"""One C3 kNN8 / fcp host-path call with FKD_PIPE_TRACE=1 (per-chunk timeline on stderr)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_12859_b200 as fk
m, dim = 10_000_000, 3
tree = fk.build_tree(fk.clustered_points(1, 1, m, dim))
qs = fk.clustered_points(1, 2, m, dim)
hq = fk.LIB.fkd_host_alloc(qs.nbytes); C.memmove(hq, qs.ctypes.data, qs.nbytes)
for kind, k in (("fcp", 1), ("knn", 8)):
    hc = fk.LIB.fkd_host_alloc(m * 4); hh = fk.LIB.fkd_host_alloc(m * k * 8)
    o = fk.BatchOptions(kind=fk.QueryKind[kind], k=k).to_c()
    for rep in range(3):
        if rep == 2: os.environ["FKD_PIPE_TRACE"] = "1"; print(kind, flush=True)
        fk.LIB.fkd_run_batch(tree.handle, hq, m, dim, C.byref(o), hc, hh, None)
        sys.stderr.flush()
    os.environ.pop("FKD_PIPE_TRACE", None)
