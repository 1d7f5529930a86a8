"""Run encode(EdgeList) of one BASELINE config on cuda:0 `reps` times (for
ncu captures: every launch of the pipeline appears once per rep).

  python tools/encode_once.py CONFIG [REPS] [--fp32] [--no-stream]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2406_03726_b200 as G  # noqa: E402
from paper_2406_03726_b200 import _lib, synth  # noqa: E402

cfg = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 2
if "--no-stream" in sys.argv:
    _lib.load().gee_debug_set(_lib.DEBUG_STREAM, 1)
for a in sys.argv:
    if a.startswith("--nt="):
        _lib.load().gee_debug_set(6, int(a[5:]))
    if a.startswith("--tile="):
        _lib.load().gee_debug_set(_lib.DEBUG_STREAM_TILE, int(a[7:]))
c = synth.make_config(cfg, "cuda")
edges = G.EdgeList(c["n"], c["rows"], c["cols"], c["weights"], c["directed"])
_, w = edges.weight_kind()
f = c["flags"]
enc = G.GeeEncoder(c["n"], c["e"], c["k"], c["directed"], G.EmbedOptions(bool(f & 1), bool(f & 2), bool(f & 4)),
                   "cuda", nonneg=bool(edges.nonneg),
                   dtype=torch.float32 if "--fp32" in sys.argv else torch.float64)
for _ in range(reps):
    enc.run(edges.rows, edges.cols, w, c["labels"], check=True)
torch.cuda.synchronize()
print("ok", cfg, c["n"], c["e"])
