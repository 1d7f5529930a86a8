"""Probe: CUDA-graph capture of the encode pipeline with per-kernel event nodes."""
import ctypes
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2406_03726_b200 as G  # noqa: E402
from paper_2406_03726_b200 import _lib, synth  # noqa: E402

c = synth.make_config(1)
dev = torch.device("cuda")
rows = torch.as_tensor(c["rows"], device=dev)
cols = torch.as_tensor(c["cols"], device=dev)
lab = torch.as_tensor(c["labels"], device=dev)
enc = G.GeeEncoder(c["n"], c["e"], 3, False, G.EmbedOptions(True, True, True))
lib = _lib.load()
enc.capture(rows, cols, None, lab, profile=True)
enc.replay()
torch.cuda.synchronize()
ms = (ctypes.c_float * 64)()
nm = (ctypes.c_char_p * 64)()
got = lib.gee_profile_read(ms, nm, 64)
print("got", got, lib.gee_last_error_string())
for j in range(max(got, 0)):
    print(nm[j], ms[j])
