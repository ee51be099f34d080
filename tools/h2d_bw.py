"""Pinned host -> device copy bandwidth: one stream vs split across copy streams."""
import torch

n = 4 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(3):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        cur = torch.cuda.current_stream()
        step = n // ns
        for i, s in enumerate(streams):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
        for s in streams:
            cur.wait_stream(s)
        b.record()
        torch.cuda.synchronize()
    print(f"{ns} stream(s): {n / a.elapsed_time(b) / 1e6:.1f} GB/s", flush=True)
hd = torch.empty(n, dtype=torch.uint8).pin_memory()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
hd.copy_(d, non_blocking=True)
b.record()
torch.cuda.synchronize()
print(f"D2H: {n / a.elapsed_time(b) / 1e6:.1f} GB/s")
