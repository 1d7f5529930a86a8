"""Per-step timeline of k_bm_gemm CTA 0 (build with -DGEE_TRACE; debug only)."""
import ctypes
import numpy as np
import torch
import paper_2406_03726_b200 as G
from paper_2406_03726_b200 import synth, _lib

c = synth.make_config(1)
dev = torch.device("cuda")
rows = torch.as_tensor(c["rows"], device=dev)
cols = torch.as_tensor(c["cols"], device=dev)
lab = torch.as_tensor(c["labels"], device=dev)
enc = G.GeeEncoder(c["n"], c["e"], 3, False, G.EmbedOptions(True, True, True))
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
for _ in range(5):
    flush.zero_()
    enc.run(rows, cols, None, lab)
torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_ulonglong * (10 * 64 + 160 + 1920))()
assert lib.gee_trace_dump(buf) == 0
arr = np.array(buf, dtype=np.int64); t = arr[:640].reshape(10, 64); ends = arr[640:640 + 148]
t0 = t[7, 0]
print("start->rep", t[7, 1] - t0, "->setup", t[7, 2] - t0, "rep: pre", t[7, 3] - t0, "loaded", t[7, 4] - t0, "flag", t[7, 5] - t0)
print("step tma  exp0  exp1  exp2  exp3  mma")
for i in range(48):
    print(i, *[f"{(t[s, i] - t0) if t[s, i] else -1:>7}" for s in (0, 1, 2, 3, 4, 8)])
print("epi acc ready", t[9, 0] - t0, t[9, 1] - t0, "epi done", t[9, 8] - t0, t[9, 9] - t0)
for seg in range(3):
    print("seg", seg, "tmem", t[9, 16 + 8 * seg] - t0, "store+fence", t[9, 17 + 8 * seg] - t0, "atomic", t[9, 18 + 8 * seg] - t0,
          "merged", t[9, 19 + 8 * seg] - t0, "z", t[9, 20 + 8 * seg] - t0)
# a finishing CTA: look at CTA traces only for CTA 0
print("cta end: min", (ends.min() - t0), "max", (ends.max() - t0), "argmax", ends.argmax())
cta = arr[800:800 + 1920].reshape(160, 12)[:148]
b0 = cta[:, 0].min()
for j, nm in enumerate(["entry", "setup", "last_mma", "epi_done", "seg0_acc", "seg0_pub", "step0_exp", "-", "polled", "merged", "z_done", "last_acc"]):
    v = (cta[:, j] - b0) / 1e3
    print(f"{nm:>9} us: min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f}")
v = (ends - b0) / 1e3
print(f"{'end':>9} us: min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f}")
for b in range(6):
    print("cta", b, " ".join(f"{(cta[b, j] - b0) / 1e3:7.2f}" if cta[b, j] else "   -   " for j in range(12)))
