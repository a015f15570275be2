"""fkd_run_batch with pinned vs pageable (plain numpy) host buffers, C3 (development aid)."""
import ctypes as C, json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_12859_b200 as fk

m, dim = 10_000_000, 3
tree = fk.build_tree(fk.clustered_points(1, 1, m, dim))
qs = fk.clustered_points(1, 2, m, dim)
hq = fk.LIB.fkd_host_alloc(qs.nbytes); C.memmove(hq, qs.ctypes.data, qs.nbytes)
for kind, k in (("fcp", 1), ("knn", 8)):
    o = fk.BatchOptions(kind=fk.QueryKind[kind], k=k).to_c()
    hc = fk.LIB.fkd_host_alloc(m * 4); hh = fk.LIB.fkd_host_alloc(m * k * 8)
    pc = np.empty(m, np.int32); ph = np.empty(m * k, np.int64)
    pc.fill(0); ph.fill(0)  # touch the pages
    rec = {"kind": kind}
    for name, (qa, ca, ha) in (("pinned", (hq, hc, hh)),
                               ("pageable", (qs.ctypes.data, pc.ctypes.data, ph.ctypes.data)),
                               ("pageable_direct", (qs.ctypes.data, pc.ctypes.data, ph.ctypes.data))):
        os.environ["FKD_PAGEABLE_STAGING"] = "0" if name == "pageable_direct" else "1"
        ts = []
        for rep in range(4):
            t = time.perf_counter()
            rc = fk.LIB.fkd_run_batch(tree.handle, C.c_void_p(qa), m, dim, C.byref(o), C.c_void_p(ca), C.c_void_p(ha), None)
            ts.append(time.perf_counter() - t)
            assert rc == 0, fk.LIB.fkd_last_error()
        rec[name + "_ms"] = round(min(ts[1:]) * 1e3, 2)
    pinc = np.ctypeslib.as_array(C.cast(hc, C.POINTER(C.c_int32)), shape=(m,))
    pinh = np.ctypeslib.as_array(C.cast(hh, C.POINTER(C.c_int64)), shape=(m * k,))
    rec["equal"] = bool(np.array_equal(pinc, pc) and np.array_equal(pinh, ph))
    print(json.dumps(rec), flush=True)
    fk.LIB.fkd_host_free(hc); fk.LIB.fkd_host_free(hh)
