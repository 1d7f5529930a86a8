"""Time the reference's own numba pipeline beside its C restatement (build
container only: it imports /root/reference, which never travels to the GPU box).

For each BASELINE config: the same host arrays both bench arms use
(oracle/gee_gen.c), the reference timed region `encode(EdgeList(...).to_csr(),
LabelVector, EmbedOptions)` (cli.py:170-180) after `_kernels.warmup()`
(cli.py:192), then the C port (oracle/gee_oracle.c) on the same arrays, 1
thread each, and the max |dZ| between the two.  One JSON line per config.

  python tools/time_numba_reference.py [CONFIGS...] [--sample-edges S] [--repeats R]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import graphee  # noqa: E402
from graphee import _kernels  # noqa: E402
from graphee.embedding import EmbedOptions, LabelVector, encode  # noqa: E402
from graphee.graph_io import EdgeList  # noqa: E402

import bench  # noqa: E402
from oracle import oracle as O  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="*", type=int, default=[0, 1, 2, 4, 3])
ap.add_argument("--sample-edges", type=int, default=1 << 25, help="configs[3]: time the first S edges")
ap.add_argument("--repeats", type=int, default=2)
args = ap.parse_args()

_kernels.warmup()
print(json.dumps({"numba": _kernels.NUMBA_ENABLED, "graphee": getattr(graphee, "__version__", "?"),
                  "threads": 1, "host_cpus": os.cpu_count()}), flush=True)
for idx in args.configs:
    c = bench.load_config(idx, "cpu")
    rows, cols, w, labels = bench.host_arrays(c)
    sample = None
    if idx == 3 and args.sample_edges and args.sample_edges < rows.shape[0]:
        sample = args.sample_edges
        rows, cols, w = rows[:sample], cols[:sample], w[:sample]
    f = c["flags"]
    opts = EmbedOptions(laplacian=bool(f & 1), diagonal=bool(f & 2), correlation=bool(f & 4))
    lv = LabelVector(np.asarray(labels, np.int64), c["k"])
    edges = EdgeList(c["n"], rows, cols, w, c["directed"])
    tn, z = [], None
    for _ in range(args.repeats):
        t0 = time.perf_counter()
        z = encode(edges.to_csr(), lv, opts)
        tn.append(time.perf_counter() - t0)
    tc, zc = [], None
    for _ in range(args.repeats):
        t0 = time.perf_counter()
        st, zc, _ = O.encode_edges(rows, cols, np.asarray(w, np.float64), c["n"], c["directed"], labels, c["k"], f)
        tc.append(time.perf_counter() - t0)
    e = int(rows.shape[0])
    line = {"config": idx, "workload": c.get("name", str(idx)), "n_edges": e,
            "sample": f"first {sample} edges" if sample else "full",
            "numba_s": tn, "numba_edges_per_s": e / min(tn),
            "c_port_s": tc, "c_port_edges_per_s": e / min(tc),
            "max_abs_dz_numba_vs_port": float(np.max(np.abs(z - zc))) if z.size else 0.0}
    print(json.dumps(line), flush=True)
    del edges, z, zc
