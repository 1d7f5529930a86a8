#!/usr/bin/env python3
"""Generate tests/golden/reference_extra.npz by running the REFERENCE itself
(build container only; the GPU box reads only the .npz):

    python tests/golden/make_extra_golden.py

Over the same seeded inputs as make_golden.py it records
* build_weight_matrix(labels)        (embedding.py:92-107)
* encode_reference(edges, labels, o) for all 8 option combos, or the
  exception class it raised          (embedding.py:146-200)
* CsrMatrix.from_triplets of the raw triplets as an n x n and as a
  rectangular n x (n + 3) matrix     (sparse.py:33-68: duplicates summed in
  input order, exact zeros dropped)
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import REF_SRC, cases  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_extra.npz")


def main():
    sys.path.insert(0, REF_SRC)
    import graphee
    from graphee import CsrMatrix, EdgeList, EmbedOptions, LabelVector, build_weight_matrix, encode_reference

    rng = np.random.default_rng(20240606)  # the same draws as reference_cases.npz
    store, names = {}, []
    for idx, (name, n, rows, cols, w, directed, labels, k) in enumerate(cases(rng)):
        p = f"c{idx}_"
        names.append(name)
        rows, cols = np.asarray(rows, np.int64), np.asarray(cols, np.int64)
        w, labels = np.asarray(w, np.float64), np.asarray(labels, np.int64)
        store[p + "meta"] = np.array([n, k, int(directed)], np.int64)
        store[p + "rows"], store[p + "cols"], store[p + "w"], store[p + "labels"] = rows, cols, w, labels
        lv = LabelVector(labels, k)
        wm = build_weight_matrix(lv)
        store[p + "wm_indptr"], store[p + "wm_cols"], store[p + "wm_vals"] = wm.index_pointers, wm.col_indices, wm.data
        edges = EdgeList(n, rows, cols, w, directed)
        for opts in EmbedOptions.all_combinations():
            tag = f"r{int(opts.laplacian)}{int(opts.diagonal)}{int(opts.correlation)}"
            try:
                store[p + tag] = encode_reference(edges, lv, opts)
            except graphee.GrapheeError as ex:
                store[p + tag + "_error"] = np.array(type(ex).__name__)
        for tag, nc in (("ft", n), ("ftr", n + 3)):
            m = CsrMatrix.from_triplets(rows, cols, w, n, nc)
            store[p + tag + "_indptr"], store[p + tag + "_cols"], store[p + tag + "_vals"] = (
                m.index_pointers, m.col_indices, m.data)
    store["names"] = np.array(names)
    store["generator"] = np.array(f"graphee {graphee.__version__} via {REF_SRC}; numpy {np.__version__}")
    np.savez_compressed(OUT, **store)
    print(f"wrote {OUT}: {len(names)} cases, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
