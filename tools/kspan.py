"""Kernel spans of the bitmap pipeline on configs[1] (GEE_TRACE build; debug only).

Prints, relative to k_bm_set's first CTA: each kernel's first CTA start,
last dependency-wait release and last CTA end, for one encode after an L2 flush."""
import ctypes
import sys
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
lib = _lib.load()
lib.gee_kspan.argtypes = [ctypes.c_void_p, ctypes.c_int]
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
g = torch.cuda.CUDAGraph()
for _ in range(3):
    enc.run(rows, cols, None, lab, check=False)
torch.cuda.synchronize()
with torch.cuda.graph(g):
    enc.run(rows, cols, None, lab, check=False)
names = ["k_bm_set", "k_bm_sym", "k_bm_table", "k_bm_gemm"]
noflush = len(sys.argv) > 1 and sys.argv[1] == 'noflush'
for rep in range(3):
    if not noflush:
        flush.zero_()
    torch.cuda.synchronize()
    lib.gee_kspan(None, 1)
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    t.record()
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 24)()
    lib.gee_kspan(ctypes.addressof(buf), 0)
    a = np.array(buf, dtype=np.uint64).reshape(8, 3).astype(np.int64)
    t0 = a[0, 0]
    print(f"replay {rep}: {s.elapsed_time(t) * 1e3:.1f} us (events)")
    for k, nm in enumerate(names):
        w = (a[k, 1] - t0) / 1e3 if a[k, 1] < (1 << 62) else float("nan")
        print(f"  {nm:>11}: start {(a[k, 0] - t0) / 1e3:7.2f}  dep {w:7.2f}  end {(a[k, 2] - t0) / 1e3:7.2f}")
