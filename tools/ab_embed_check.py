"""Compare Z of the stream embed variants (debug knob 6) on BASELINE configs:
  python tools/ab_embed_check.py NT_A NT_B CONFIG...
prints the max entrywise |Za - Zb| / max(|Za row|) per config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2406_03726_b200 as G  # noqa: E402
from paper_2406_03726_b200 import _lib, synth  # noqa: E402

lib = _lib.load()
na, nb = int(sys.argv[1]), int(sys.argv[2])
for cfg in [int(x) for x in sys.argv[3:]]:
    c = synth.make_config(cfg, "cuda")
    edges = G.EdgeList(c["n"], c["rows"], c["cols"], c["weights"], c["directed"])
    lab = G.LabelVector(c["labels"], c["k"])
    f = c["flags"]
    opts = G.EmbedOptions(bool(f & 1), bool(f & 2), bool(f & 4))
    out = []
    for nt in (na, nb):
        lib.gee_debug_set(6, nt)
        for dt in (torch.float64, torch.float32):
            out.append(torch.as_tensor(G.encode(edges, lab, opts, dtype=dt), device="cuda").double())
    for i, name in ((0, "f64"), (1, "f32")):
        za, zb = out[i], out[i + 2]
        scale = za.abs().amax(dim=1, keepdim=True).clamp_min(1e-300)
        print(f"cfg{cfg} {name}: max rel diff {((za - zb).abs() / scale).max().item():.3e}", flush=True)
    del out
lib.gee_debug_set(6, 128)
