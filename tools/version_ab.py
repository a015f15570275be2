"""Same-box A/B of whole library versions (package + .so at another root,
e.g. a git worktree under build/): C3 step, serial calls and, where the
version has it, one run_batches_device submission.
    python tools/version_ab.py <root> [<root> ...]"""
import os
import subprocess
import sys

CODE = r'''
import sys, numpy as np, torch
sys.path.insert(0, ROOT)
import paper_2210_12859_b200 as fk
dev = torch.device("cuda", 0)
n = m = 10_000_000
nodes = fk.build_level_order_device(torch.from_numpy(fk.clustered_points(1, 1, n, 3)).to(dev))
tree = fk.KdTree.from_device(nodes)
q = torch.from_numpy(fk.clustered_points(1, 2, m, 3)).to(dev)
outs = [(torch.empty(m, dtype=torch.int32, device=dev), torch.empty(m, dtype=torch.int64, device=dev)),
        (torch.empty(m, dtype=torch.int32, device=dev), torch.empty(m * 8, dtype=torch.int64, device=dev))]
opts = [fk.BatchOptions(kind=fk.QueryKind.fcp), fk.BatchOptions(kind=fk.QueryKind.knn, k=8)]
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
st = torch.cuda.current_stream()
modes = ["serial"] + (["concurrent"] if hasattr(fk, "run_batches_device") else [])
for mode in modes:
    def step():
        if mode == "serial":
            for (c, h), o in zip(outs, opts):
                fk.run_batch_device(tree, q, c, h, o, stream=st)
        else:
            fk.run_batches_device(tree, [(q, c, h, o) for (c, h), o in zip(outs, opts)], stream=st)
    for _ in range(3): step()
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); step(); e1.record(st); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{ROOT} {mode} ms/step {np.mean(ts):.3f}", flush=True)
'''

for rep in range(2):
    for root in sys.argv[1:]:
        subprocess.run([sys.executable, "-c", f"ROOT = {os.path.abspath(root)!r}\n" + CODE], check=False)
