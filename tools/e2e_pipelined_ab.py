"""C3 serving loop through fkd_submit_batches / fkd_wait (fcp + kNN8 per step,
pinned buffers, `depth` jobs in flight) under knob variants; the synchronous
fkd_run_batches call is the depth-1 row.
    python tools/e2e_pipelined_ab.py '' 'FKD_CHUNK_DIV=4' ..."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_12859_b200 as fk  # noqa: E402

m, dim, steps = 10_000_000, 3, 10
tree = fk.build_tree(fk.clustered_points(1, 1, m, dim))
qs = fk.clustered_points(1, 2, m, dim)
hq = fk.LIB.fkd_host_alloc(qs.nbytes)
C.memmove(hq, qs.ctypes.data, qs.nbytes)
opts = (fk.BatchOptions(kind=fk.QueryKind.knn, k=8), fk.BatchOptions())
sets = []
for _ in range(3):
    arr = (fk._lib.fkd_host_batch * 2)()
    for i, o in enumerate(opts):
        arr[i].queries, arr[i].m, arr[i].dim, arr[i].opt = hq, m, dim, o.to_c()
        arr[i].counts, arr[i].hits = fk.LIB.fkd_host_alloc(m * 4), fk.LIB.fkd_host_alloc(m * o.stride * 8)
    sets.append(arr)


def run(depth, n):
    pending = []
    for s in range(n):
        h = C.c_void_p()
        assert fk.LIB.fkd_submit_batches(tree.handle, sets[s % depth], 2, C.byref(h)) == 0
        pending.append(h)
        if len(pending) == depth:
            assert fk.LIB.fkd_wait(pending.pop(0)) == 0
    for h in pending:
        assert fk.LIB.fkd_wait(h) == 0


for v in sys.argv[1:] or [""]:
    env = dict(p.split("=", 1) for p in v.split(";") if p)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    for depth in (1, 2, 3):
        run(depth, 3)
        t0 = time.perf_counter()
        run(depth, steps)
        ms = (time.perf_counter() - t0) / steps * 1e3
        print(f"{v or 'default':40s} depth {depth}: {ms:6.2f} ms/step ({2 * m / ms / 1e6:.3f} G q/s)", flush=True)
    for k_, v_ in old.items():
        if v_ is None:
            os.environ.pop(k_, None)
        else:
            os.environ[k_] = v_
