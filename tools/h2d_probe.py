"""Pinned host->device copy bandwidth: one large copy vs chunks over 1-4 streams (dev tool)."""
import torch

n = 1 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for streams in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    for chunk in (n, n // 8, n // 64):
        best = 1e9
        for _ in range(3):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i, o in enumerate(range(0, n, chunk)):
                s = ss[i % streams]
                s.wait_event(e0)
                with torch.cuda.stream(s):
                    d[o:o + chunk].copy_(h[o:o + chunk], non_blocking=True)
            for s in ss:
                e1.wait_stream(s) if hasattr(e1, "wait_stream") else torch.cuda.current_stream().wait_stream(s)
            torch.cuda.current_stream().wait_stream(ss[0])
            for s in ss:
                torch.cuda.current_stream().wait_stream(s)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(f"streams {streams} chunk {chunk >> 20:5d} MB: {n / best / 1e6:.1f} GB/s")
