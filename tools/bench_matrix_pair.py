"""The same Table-1 style grid through the B200 path and the reference
(flatkd::run_bench_matrix + write_bench_csv from oracle/_ref, all host
threads), written side by side under profiles/: rows diff on every column
but engine/threads/timings.  Usage: python tools/bench_matrix_pair.py <tag>"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import Reference  # noqa: E402
from paper_2210_12859_b200 import QueryKind  # noqa: E402
from paper_2210_12859_b200 import bench_matrix as bm  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
out = os.path.join("profiles", tag)
os.makedirs(out, exist_ok=True)
INF = float("inf")
grid = [("fcp", (8,), (INF,)), ("knn", (1, 4, 8, 16), (INF, 0.01))]
ref = Reference()
with open(os.path.join(out, "bench_matrix_b200.csv"), "w") as fb, \
        open(os.path.join(out, "bench_matrix_reference.csv"), "w") as fr:
    for i, (kind, ks, rs) in enumerate(grid):
        base = bm.BenchConfig(n_queries=1_000_000, k_dim=3, kind=QueryKind[kind], reps=3)
        rows = bm.run_bench_matrix(base, [1_000_000, 10_000_000], ks, rs)
        import io
        buf = io.StringIO()
        bm.write_bench_csv(buf, rows)
        text = buf.getvalue()
        rtext = ref.bench_matrix_csv(1_000_000, 3, kind, 3, [1_000_000, 10_000_000], ks, rs)
        fb.write(text if i == 0 else text.split("\n", 1)[1])
        fr.write(rtext if i == 0 else rtext.split("\n", 1)[1])
        print(text, rtext, flush=True)
