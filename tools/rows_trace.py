"""Slowest per-row tasks (tiers X and B) of k_rows on a config (GEE_TRACE build; debug only)."""
import ctypes, sys
import numpy as np
import torch
import paper_2406_03726_b200 as G
from paper_2406_03726_b200 import _lib, synth
cfg = int(sys.argv[1])
c = synth.make_config(cfg, device="cuda" if cfg in (3, 4) else "cpu")
dev = torch.device("cuda")
rows = torch.as_tensor(c["rows"], device=dev); cols = torch.as_tensor(c["cols"], device=dev)
w = torch.as_tensor(c["weights"], device=dev)
if bool((w == 1.0).all()):
    w = None
lab = torch.as_tensor(c["labels"], device=dev)
f = c["flags"]
enc = G.GeeEncoder(c["n"], c["e"], c["k"], c["directed"], G.EmbedOptions(bool(f & 1), bool(f & 2), bool(f & 4)))
enc.run(rows, cols, w, lab); torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_ulonglong * (4096 * 3))(); n = ctypes.c_uint(0)
lib.gee_rows_dump(buf, ctypes.byref(n))
enc.run(rows, cols, w, lab); torch.cuda.synchronize()
lib.gee_rows_dump(buf, ctypes.byref(n))
t = np.array(buf, dtype=np.uint64).reshape(4096, 3)[: min(n.value, 4096)]
print("tasks", n.value)
o = np.argsort(-t[:, 2].astype(np.int64))
for i in o[:12]:
    print("tier", t[i, 0], "row", t[i, 1], "cycles", t[i, 2])
