"""Pinned copy bandwidth: H2D alone, D2H alone, both at once on two streams, and
D2H while a kernel-heavy stream runs (development aid)."""
import json, time, torch
n = 1 << 30
h1 = torch.empty(n // 4, dtype=torch.float32).pin_memory(); d1 = torch.empty(n // 4, dtype=torch.float32, device="cuda")
h2 = torch.empty(n // 4, dtype=torch.float32).pin_memory(); d2 = torch.empty(n // 4, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h, reps=5):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); return n * reps / (time.perf_counter() - t) / 1e9
run(True, True, 1)
print(json.dumps({"h2d": run(True, False), "d2h": run(False, True), "bidir_each": run(True, True)}))
# D2H in 80 MB pieces (the pipeline's chunk size)
piece = 80 << 20
torch.cuda.synchronize(); t = time.perf_counter()
for r in range(5):
    for off in range(0, n - piece, piece):
        with torch.cuda.stream(s2): h2[off // 4:(off + piece) // 4].copy_(d2[off // 4:(off + piece) // 4], non_blocking=True)
torch.cuda.synchronize(); print(json.dumps({"d2h_80MB_pieces": 5 * (n - piece) // piece * piece / (time.perf_counter() - t) / 1e9}))
