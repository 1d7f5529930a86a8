"""Small end-to-end workload for compute-sanitizer (one tool per run):
every kernel family once -- generators, the stream encode (unit / f32 / f64,
split buckets), the CSR assembly paths + embed, the bitmap path, the text
parser -- on graphs small enough for the sanitizer's slowdown."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_03726_b200 as G  # noqa: E402
from paper_2406_03726_b200 import _lib, synth, textio  # noqa: E402

lib = _lib.load()
rng = np.random.default_rng(1)
opts = G.EmbedOptions(True, True, True)
for idx, sd in ((0, 0), (2, 6), (3, 10), (4, 8)):
    c = synth.make_config(idx, "cuda", sd)
    e = G.EdgeList(c["n"], c["rows"], c["cols"], c["weights"], c["directed"])
    lab = G.LabelVector(c["labels"], c["k"])
    G.encode(e, lab, opts)
    G.encode(e, lab, opts, dtype=torch.float32)
    for force in (1, 2, 3):  # the CSR assembly paths (stream off)
        lib.gee_debug_set(_lib.DEBUG_FORCE_BUCKETS, force)
        lib.gee_debug_set(_lib.DEBUG_STREAM, 1)
        csr = e.to_csr()
        G.encode(e, lab, opts)
        G.degree_vector(csr, diagonal=True)
        lib.gee_debug_set(_lib.DEBUG_FORCE_BUCKETS, 0)
        lib.gee_debug_set(_lib.DEBUG_STREAM, 0)
# split buckets in the stream path
n, m = 20000, 200000
rows = rng.integers(0, n, m)
rows[: m // 2] = 3
G.encode(G.EdgeList(n, rows, rng.integers(0, n, m), 1.0 - rng.random(m)), G.LabelVector(rng.integers(-1, 50, n), 50),
         opts)
text = "".join(f"{i} {j} {float(w)!r}\n" for i, j, w in zip(rng.integers(0, 99, 500), rng.integers(0, 99, 500), rng.random(500)))
textio.parse_edge_list(text)
textio.parse_labels("".join(f"{i} {i % 3}\n" for i in range(99)))
torch.cuda.synchronize()
print("sanitize case ok")
