#!/usr/bin/env python3
"""Generate tests/golden/reference_cases.npz by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package `graphee` from /root/reference/pkg/src and
records, for seeded random graphs (directed and undirected, weighted, with
duplicates, self-loops, negative weights, unlabeled nodes) plus the
reference tests' hand cases:

* the to_csr() result   (graph_io.py:78-92 -> _kernels.coo_to_csr)
* add_identity()        (sparse.py:184-190)
* degree_vector() of A and of A+I  (sparse.py:193-196)
* laplacian_normalize() (sparse.py:199-226) or the error it raises
* class_counts()        (embedding.py:68-71)
* encode() for all 8 EmbedOptions combos (embedding.py:110-131), or the
  exception class it raised

The fixture file is small and committed; the GPU box never sees the
reference (tests read only the .npz).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_cases.npz")


def cases(rng):
    """Seeded fuzz inputs: (name, n, rows, cols, w, directed, labels, k)."""
    out = []
    # hand cases from the reference tests (test_embedding.py:20-23, :107-114, :233-240)
    out.append(("triangle", 3, [0, 0, 1], [1, 2, 2], [1.0, 1.0, 1.0], False, [0, 1, 1], 2))
    out.append(("single_edge", 2, [0], [1], [1.0], False, [0, 1], 2))
    out.append(("edgeless", 4, [], [], [], False, [0, 1, 0, 1], 2))
    out.append(("all_unlabeled", 3, [0, 0, 1], [1, 2, 2], [1.0, 1.0, 1.0], False, [-1, -1, -1], 2))
    out.append(("unlabeled_middle", 3, [0, 1], [1, 2], [1.0, 1.0], False, [0, -1, 0], 1))
    out.append(("empty_classes", 3, [0, 1], [1, 2], [1.0, 1.0], False, [2, 2, 2], 3))
    # cancelling duplicates, -1 self loop (cancels under A+I), negative degree
    out.append(("cancel_dup", 4, [0, 0, 1, 2, 3], [1, 1, 2, 2, 0], [1.5, -1.5, 2.0, -1.0, 0.25],
                False, [0, 1, 0, 1], 2))
    out.append(("neg_degree", 2, [0], [1], [-2.0], False, [0, 1], 2))
    out.append(("triple_dup", 3, [0, 0, 0, 1], [1, 1, 1, 2], [0.1, 0.2, 0.3, 1e-17], True,
                [0, 1, 1], 2))
    for t in range(60):
        n = int(rng.integers(2, 120))
        k = int(rng.integers(1, 7))
        m = int(rng.integers(0, 4 * n + 1))
        rows = rng.integers(0, n, m)
        cols = rng.integers(0, n, m)
        kind = t % 4
        if kind == 0:
            w = 2.0 * (1.0 - rng.random(m))          # (0, 2]
        elif kind == 1:
            w = np.ones(m)                           # unit weights
        elif kind == 2:
            w = rng.uniform(-2.0, 2.0, m)            # signed
        else:
            w = rng.choice([-1.0, 0.5, 1.0, 2.0, 3.0], m)  # small dyadic values
        if m >= 3 and t % 5 == 0:
            # force a 3-run of duplicates so the in-order sum matters
            rows[1:3] = rows[0]
            cols[1:3] = cols[0]
        labels = rng.integers(0, k, n)
        labels[rng.random(n) < 0.2] = -1
        out.append((f"fuzz{t}", n, rows, cols, w, bool(t % 2), labels, k))
    # two larger weighted multigraphs (long duplicate runs, hub rows)
    for t in range(2):
        n = 500
        m = 5000
        hub = rng.integers(0, n, 5)
        rows = np.where(rng.random(m) < 0.2, rng.choice(hub, m), rng.integers(0, n, m))
        cols = rng.integers(0, n // 3, m)
        w = 1.0 - rng.random(m)
        labels = rng.integers(0, 5, n)
        labels[rng.random(n) < 0.1] = -1
        out.append((f"multi{t}", n, rows, cols, w, bool(t), labels, 5))
    return out


def main():
    sys.path.insert(0, REF_SRC)
    import graphee
    from graphee import (EdgeList, EmbedOptions, LabelVector, add_identity, degree_vector,
                         encode, laplacian_normalize)

    rng = np.random.default_rng(20240606)
    store = {}
    names = []
    for idx, (name, n, rows, cols, w, directed, labels, k) in enumerate(cases(rng)):
        p = f"c{idx}_"
        names.append(name)
        rows = np.asarray(rows, np.int64)
        cols = np.asarray(cols, np.int64)
        w = np.asarray(w, np.float64)
        labels = np.asarray(labels, np.int64)
        store[p + "meta"] = np.array([n, k, int(directed)], np.int64)
        store[p + "rows"], store[p + "cols"], store[p + "w"] = rows, cols, w
        store[p + "labels"] = labels
        edges = EdgeList(n, rows, cols, w, directed)
        lv = LabelVector(labels, k)
        adj = edges.to_csr()
        store[p + "csr_indptr"] = adj.index_pointers
        store[p + "csr_cols"] = adj.col_indices
        store[p + "csr_vals"] = adj.data
        aug = add_identity(adj)
        store[p + "aug_indptr"] = aug.index_pointers
        store[p + "aug_cols"] = aug.col_indices
        store[p + "aug_vals"] = aug.data
        store[p + "deg"] = degree_vector(adj)
        store[p + "deg_aug"] = degree_vector(aug)
        try:
            lap = laplacian_normalize(adj, degree_vector(adj))
            store[p + "lap_indptr"] = lap.index_pointers
            store[p + "lap_cols"] = lap.col_indices
            store[p + "lap_vals"] = lap.data
        except graphee.NumericalDomainError:
            store[p + "lap_error"] = np.array(1)
        store[p + "counts"] = lv.class_counts()
        for opts in EmbedOptions.all_combinations():
            tag = f"z{int(opts.laplacian)}{int(opts.diagonal)}{int(opts.correlation)}"
            try:
                store[p + tag] = encode(adj, lv, opts)
            except graphee.GrapheeError as ex:
                store[p + tag + "_error"] = np.array(type(ex).__name__)
    store["names"] = np.array(names)
    store["generator"] = np.array(f"graphee {graphee.__version__} via {REF_SRC}; numpy {np.__version__}")
    np.savez_compressed(OUT, **store)
    print(f"wrote {OUT}: {len(names)} cases, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
