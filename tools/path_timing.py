"""Time gee_encode_edges on one config with a forced K2 path (debug tool).

usage: PYTHONPATH=. python tools/path_timing.py CONFIG MODE   (MODE 0 default, 1 buckets, 2 no bitmap)
"""
import sys

import torch

import paper_2406_03726_b200 as G
from paper_2406_03726_b200 import _lib, synth

cfg, mode = int(sys.argv[1]), int(sys.argv[2])
c = synth.make_config(cfg, device="cuda" if cfg in (3, 4) else "cpu")
dev = torch.device("cuda")
rows = torch.as_tensor(c["rows"], device=dev)
cols = torch.as_tensor(c["cols"], device=dev)
w = torch.as_tensor(c["weights"], device=dev)
if bool((w == 1.0).all()):
    w = None
lab = torch.as_tensor(c["labels"], device=dev)
lib = _lib.load()
lib.gee_debug_set(_lib.DEBUG_FORCE_BUCKETS, mode)
f = c["flags"]
enc = G.GeeEncoder(c["n"], c["e"], c["k"], c["directed"], G.EmbedOptions(bool(f & 1), bool(f & 2), bool(f & 4)))
for _ in range(3):
    enc.run(rows, cols, w, lab)
torch.cuda.synchronize()
s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    enc.run(rows, cols, w, lab)
t.record()
torch.cuda.synchronize()
ms = s.elapsed_time(t) / 10
print(f"cfg{cfg} mode{mode}: {ms:.3f} ms/encode, {c['e'] / ms / 1e6:.2f} G edges/s")
