"""Pure-write vs copy HBM bandwidth on this GPU (torch fill_ / copy_), for the
write-bound embed roofline (configs[4] writes an 8 GB Z)."""
import torch

z = torch.empty(1_000_000_000, dtype=torch.float64, device="cuda")  # 8 GB
src = torch.empty(500_000_000, dtype=torch.float64, device="cuda")
dst = torch.empty_like(src)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn, nbytes in [("fill 8 GB", lambda: z.fill_(1.0), 8e9),
                         ("zero 8 GB", lambda: z.zero_(), 8e9),
                         ("copy 4+4 GB", lambda: dst.copy_(src), 8e9)]:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(10):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    print(f"{name}: {ms:.3f} ms  {nbytes / ms / 1e6:.0f} GB/s")
