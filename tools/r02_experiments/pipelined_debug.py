import ctypes as C, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2210_12859_b200 as fk
m, dim = 10_000_000, 3
dev = torch.device("cuda", 0)
tree = fk.KdTree.from_device(fk.build_level_order_device(torch.from_numpy(fk.clustered_points(1, 1, m, dim)).to(dev)))
qs = fk.clustered_points(1, 2, m, dim)
opts = (fk.BatchOptions(kind=fk.QueryKind.knn, k=8), fk.BatchOptions())
if "--device" in sys.argv:
    qd = torch.from_numpy(qs).to(dev)
    outs = [(torch.empty(m, dtype=torch.int32, device=dev), torch.empty(m * o.stride, dtype=torch.int64, device=dev)) for o in opts]
    for _ in range(3):
        fk.run_batches_device(tree, [(qd, c, h, o) for (c, h), o in zip(outs, opts)])
hq = fk.LIB.fkd_host_alloc(qs.nbytes); C.memmove(hq, qs.ctypes.data, qs.nbytes)
sets = []
for _ in range(2):
    arr = (fk._lib.fkd_host_batch * 2)()
    for i, o in enumerate(opts):
        arr[i].queries, arr[i].m, arr[i].dim, arr[i].opt = hq, m, dim, o.to_c()
        arr[i].counts, arr[i].hits = fk.LIB.fkd_host_alloc(m * 4), fk.LIB.fkd_host_alloc(m * o.stride * 8)
    sets.append(arr)
for s in range(3):
    t0 = time.perf_counter(); assert fk.LIB.fkd_run_batches(tree.handle, sets[0], 2) == 0
    print("sync", round((time.perf_counter() - t0) * 1e3, 2))
pending = []; t0 = time.perf_counter(); last = t0
for s in range(14):
    h = C.c_void_p(); assert fk.LIB.fkd_submit_batches(tree.handle, sets[s % 2], 2, C.byref(h)) == 0
    pending.append(h)
    if len(pending) == 2:
        assert fk.LIB.fkd_wait(pending.pop(0)) == 0
        now = time.perf_counter(); print("pipelined step", s - 1, round((now - last) * 1e3, 2)); last = now
for h in pending: fk.LIB.fkd_wait(h)
print("total per step", round((time.perf_counter() - t0) / 14 * 1e3, 2))
