"""CTA start/compute/end timeline of k_bm_sym (build with -DGEE_TRACE; debug only)."""
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
for _ in range(5):
    enc.run(rows, cols, None, lab)
torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_ulonglong * (4096 * 3))()
assert lib.gee_sym_dump(buf) == 0
t = np.array(buf, dtype=np.int64).reshape(4096, 3)[:3240]
t0 = t[:, 0].min()
t = t - t0
print("start: min/med/max", t[:, 0].min(), np.median(t[:, 0]), t[:, 0].max())
print("mid-start: med/max", np.median(t[:, 1] - t[:, 0]), (t[:, 1] - t[:, 0]).max())
print("end-mid: med/max", np.median(t[:, 2] - t[:, 1]), (t[:, 2] - t[:, 1]).max())
print("end max", t[:, 2].max())
for q in (0.1, 0.25, 0.5, 0.75, 0.9, 1.0):
    print(q, np.quantile(t[:, 0], q), np.quantile(t[:, 2], q))
