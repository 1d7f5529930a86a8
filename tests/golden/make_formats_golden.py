#!/usr/bin/env python3
"""Generate tests/golden/formats_cases.json by running the REFERENCE's text
I/O (graph_io.py:95-305) on a fixed set of inputs.  Run in the build
container (where /root/reference exists):

    python tests/golden/make_formats_golden.py

Records, per edge-list / label text and ParseOptions, the parsed arrays or the
exception class and line number; per embedding matrix, the exact CSV bytes
write_embedding produces.  The GPU box never sees the reference."""

import io
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from graphee import graph_io as R  # noqa: E402

EDGE_TEXTS = [
    ("0 1\n0 2\n1 2\n", {}, None),
    ("1,2,0.5\n2,3\n", {"index_base": 1}, None),
    ("# comment\n\n  0 1 2.5  \n\t1 2\n# trailing\n", {}, None),
    ("0 1 0.1\n1 2 1e-300\n2 3 -4.25\n3 0 1_000.5\n", {}, None),
    ("0 1\n0 x\n", {}, None),
    ("0 1 nan\n", {}, None),
    ("0 1 inf\n", {}, None),
    ("0 1 abc\n", {}, None),
    ("0 1 2 3\n", {}, None),
    ("0\n", {}, None),
    ("0 1\n", {"index_base": 1}, None),
    ("-1 0\n", {}, None),
    ("0 5\n", {}, 4),
    ("0 1\n", {}, 7),
    ("", {}, None),
    ("# only comments\n\n", {}, 3),
    ("0 1\n", {"directed": True}, None),
    ("0,1\n1 2\n", {}, None),
    ("0 1\n1,2\n", {}, None),
    ("0 1\n", {"delimiter": "comma"}, None),
    ("0\t1\t3\n+2 0003 -0.0\n", {"default_weight": 2.0}, None),
    (" 0 , 1 , 7 \n", {}, None),
]
LABEL_TEXTS = [
    ("0\n1\n1\n", {}, None, None),
    ("0 1\n3 2\n", {}, None, None),
    ("0 1\n3 2\n", {}, None, 6),
    ("-1\n2\n-1\n", {}, None, None),
    ("-2\n", {}, None, None),
    ("0 1\n0 2\n", {}, None, None),
    ("0 1\n0 1\n", {}, None, None),
    ("0\n1 2\n", {}, 4, None),
    ("-1\n-1\n", {}, None, None),
    ("-1\n-1\n", {}, 3, None),
    ("1 0\n2 1\n", {"index_base": 1}, None, None),
    ("0 1 2\n", {}, None, None),
    ("0 5\n", {}, None, 3),
    ("x\n", {}, None, None),
    ("0\n1\n", {}, 5, None),
]
Z_CASES = [
    [[0.0, 1.0], [1.0, 0.5], [1.0, 0.5]],
    [[0.1, 1 / 3, 2 / 3], [1e16, 1e15, 123456789012345.0], [5e-324, -0.0, 1e-300]],
    [[0.7071067811865475, 0.7071067811865476], [-1.5, 2.0 ** 60], [float(np.float32(0.1)), 9007199254740993.0]],
    np.random.default_rng(0).random((4, 5)).tolist(),
    [],
]


def run(fn):
    try:
        return {"ok": fn()}
    except Exception as e:  # noqa: BLE001
        return {"error": type(e).__name__, "line": getattr(e, "line_no", None)}


def main():
    out = {"edges": [], "labels": [], "embedding": []}
    for text, opts, n in EDGE_TEXTS:
        def f():
            e = R.parse_edge_list(io.StringIO(text), R.ParseOptions(**opts), n_nodes=n)
            return {"n_nodes": int(e.n_nodes), "rows": e.rows.tolist(), "cols": e.cols.tolist(),
                    "weights": [float(x).hex() for x in e.weights], "directed": bool(e.directed)}
        out["edges"].append({"text": text, "opts": opts, "n_nodes": n, "result": run(f)})
    for text, opts, k, n in LABEL_TEXTS:
        def f():
            lv = R.parse_labels(io.StringIO(text), R.ParseOptions(**opts), k_classes=k, n_nodes=n)
            return {"labels": lv.labels.tolist(), "k_classes": int(lv.k_classes)}
        out["labels"].append({"text": text, "opts": opts, "k_classes": k, "n_nodes": n, "result": run(f)})
    for z in Z_CASES:
        arr = np.asarray(z, dtype=np.float64).reshape(len(z), len(z[0]) if len(z) else 3)
        buf = io.StringIO()
        R.write_embedding(arr, buf)
        out["embedding"].append({"z": [[float(x).hex() for x in row] for row in arr], "k": arr.shape[1],
                                 "csv": buf.getvalue()})
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "formats_cases.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(f"wrote {path}: {len(out['edges'])} edge texts, {len(out['labels'])} label texts, "
          f"{len(out['embedding'])} embeddings")


if __name__ == "__main__":
    main()
