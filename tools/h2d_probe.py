"""Pinned host -> device copy bandwidth: one stream vs two concurrent streams (debug tool)."""
import torch

n = 88 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for trial in range(3):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    d.copy_(h, non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    one = a.elapsed_time(b)
    cur = torch.cuda.current_stream()
    a.record(cur)
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d[: n // 2].copy_(h[: n // 2], non_blocking=True)
    with torch.cuda.stream(s2):
        d[n // 2:].copy_(h[n // 2:], non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)
    b.record(cur)
    torch.cuda.synchronize()
    two = a.elapsed_time(b)
    print(f"88 MiB: one stream {n / one / 1e6:.1f} GB/s, two streams {n / two / 1e6:.1f} GB/s")
