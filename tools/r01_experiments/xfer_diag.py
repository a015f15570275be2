"""Transfer floor of the kNN8 host path: chunked H2D 120 MB + D2H 680 MB over 4 streams."""
import time, torch
m = 10_000_000
hq = torch.empty(m * 3, dtype=torch.float32).pin_memory()
hh = torch.empty(m * 8 * 2, dtype=torch.int32).pin_memory()
hc = torch.empty(m, dtype=torch.int32).pin_memory()
dq = torch.empty(m * 3, dtype=torch.float32, device="cuda")
dh = torch.empty(m * 8 * 2, dtype=torch.int32, device="cuda")
dc = torch.empty(m, dtype=torch.int32, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
def run(chunks, compute=False):
    per = m // chunks
    torch.cuda.synchronize(); t = time.perf_counter()
    for c in range(chunks):
        s = streams[c % 4]
        with torch.cuda.stream(s):
            a, b = c * per, (c + 1) * per
            dq[a*3:b*3].copy_(hq[a*3:b*3], non_blocking=True)
            if compute:
                torch.cuda._sleep(int(1.26e6 * 12.6 / chunks))  # ~12.6 ms of GPU time total
            hh[a*16:b*16].copy_(dh[a*16:b*16], non_blocking=True)
            hc[a:b].copy_(dc[a:b], non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e3
for chunks in (8, 16, 32):
    run(chunks); print(chunks, "copies only ms", round(min(run(chunks) for _ in range(3)), 2), "with 12.6 ms sleep", round(min(run(chunks, True) for _ in range(3)), 2))
