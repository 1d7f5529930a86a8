"""Phase trace of the stream embed (debug variant 16 + diagnostics): clock64 totals per CTA.
Needs a library built with the trace compiled in: make -C paper_2406_03726_b200/csrc EXTRA=-DGEE_EMBED_TRACE
(the normal build leaves it out: its counters cost the embed registers it does not have).
  python tools/embed_trace.py CONFIG [--nt=128] [--tile=32]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_03726_b200 as G  # noqa: E402
from paper_2406_03726_b200 import _lib, synth  # noqa: E402

cfg = int(sys.argv[1])
lib = _lib.load()
for a in sys.argv[2:]:
    if a.startswith("--nt="):
        lib.gee_debug_set(6, int(a[5:]))
    if a.startswith("--tile="):
        lib.gee_debug_set(5, int(a[7:]))
c = synth.make_config(cfg, "cuda")
edges = G.EdgeList(c["n"], c["rows"], c["cols"], c["weights"], c["directed"])
_, w = edges.weight_kind()
f = c["flags"]
enc = G.GeeEncoder(c["n"], c["e"], c["k"], c["directed"], G.EmbedOptions(bool(f & 1), bool(f & 2), bool(f & 4)),
                   "cuda", nonneg=bool(edges.nonneg))
enc.run(edges.rows, edges.cols, w, c["labels"], check=True)
buf = (ctypes.c_ulonglong * (4096 * 8))()
lib.dbg_stream_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
lib.dbg_stream_trace_read(buf, 4096 * 8)
lib.gee_debug_set(4, 16 + int(os.environ.get("VARIANT", "16")))
enc.run(edges.rows, edges.cols, w, c["labels"], check=False)
torch.cuda.synchronize()
lib.dbg_stream_trace_read(buf, 4096 * 8)
t = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 8).astype(np.float64)
t = t[t[:, 4] > 0]
tot = t[:, :4].sum(axis=1)
print(f"CTAs {t.shape[0]}  items/CTA {t[:,4].mean():.0f}  entries/CTA {t[:,5].mean():.0f}")
if t.shape[1] >= 8:
    print("in accumulate, per item: record wait %.0f  consume %.0f  refill (gather + keys) %.0f" %
          tuple(t[:, [0, 6, 7]].mean(axis=0) / t[:, 4].mean()))
print("mean cycles per CTA: wait-K0 %.0f  accumulate %.0f  tile-barrier %.0f  epilogue %.0f  total %.0f" %
      tuple(list(t[:, :4].mean(axis=0)) + [tot.mean()]))
print("per item: wait-K0 %.0f  accumulate %.0f  barrier %.0f  epilogue %.0f" %
      tuple(t[:, :4].sum(axis=0) / t[:, 4].sum()))
print("max total %.0f  min total %.0f" % (tot.max(), tot.min()))
