"""D2H bandwidth into pinned host memory: one stream vs the copy split over
two or four streams (are several copy engines faster than one on PCIe?).
    python tools/micro/d2h_streams.py"""
import torch

MB = 1 << 20
dev = torch.device("cuda", 0)
src = torch.empty(720 * MB, dtype=torch.uint8, device=dev)
dst = torch.empty(720 * MB, dtype=torch.uint8, pin_memory=True)
hsrc = torch.empty(120 * MB, dtype=torch.uint8, pin_memory=True)
ddst = torch.empty(120 * MB, dtype=torch.uint8, device=dev)
streams = [torch.cuda.Stream() for _ in range(4)]
for piece_mb in (80, 20):
    for ns in (1, 2, 4):
        for with_h2d in (False, True):
            best = 1e9
            for _ in range(5):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for s in streams:
                    s.wait_event(e0)
                n = 720 // piece_mb
                for i in range(n):
                    s = streams[i % ns]
                    with torch.cuda.stream(s):
                        dst[i * piece_mb * MB:(i + 1) * piece_mb * MB].copy_(src[i * piece_mb * MB:(i + 1) * piece_mb * MB], non_blocking=True)
                if with_h2d:
                    with torch.cuda.stream(streams[3]):
                        ddst.copy_(hsrc, non_blocking=True)
                for s in streams:
                    e1.wait_stream(s) if hasattr(e1, "wait_stream") else None
                    torch.cuda.current_stream().wait_stream(s)
                e1.record()
                e1.synchronize()
                best = min(best, e0.elapsed_time(e1))
            print(f"piece {piece_mb} MB streams {ns} h2d {with_h2d}: {best:.2f} ms  {720 * MB / best / 1e6:.1f} GB/s D2H", flush=True)
