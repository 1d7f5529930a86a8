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
buf2 = (ctypes.c_ulonglong * (512 * 6))()
lib.gee_phase_dump(buf2)
ph = np.array(buf2, dtype=np.int64).reshape(512, 6)[:296]
d = np.diff(ph[:, :5], axis=1)
print("per-CTA phase cycles (X, D+B, M, S): mean", d.mean(axis=0).astype(int), "max", d.max(axis=0))
print("CTA total max", (ph[:, 4] - ph[:, 0]).max(), "argmax", (ph[:, 4] - ph[:, 0]).argmax())
buf3 = (ctypes.c_ulonglong * (512 * 4))()
lib.gee_lsd_dump(buf3)
ls = np.array(buf3, dtype=np.int64).reshape(512, 4)[:296]
o = np.argsort(-(ls[:, 1] + ls[:, 2]))
for i in o[:6]:
    print("CTA", i, "row", ls[i, 3], "L", ls[i, 0], "lsd cycles", ls[i, 1], "finish cycles", ls[i, 2])
buf4 = (ctypes.c_ulonglong * (512 * 8))()
lib.gee_fin_dump(buf4)
fn = np.array(buf4, dtype=np.int64).reshape(512, 8)[:296]
o = np.argsort(-fn[:, 0])
for i in o[:6]:
    print("CTA", i, "row", fn[i, 6], "L", fn[i, 0], "runs", fn[i, 1], "scan+out", fn[i, 2], "cert", fn[i, 3], "degree", fn[i, 4], "certified", fn[i, 5])
