"""INTEGRATION.md's reference-side ctypes binding, executed verbatim, and
encode() on duck-typed reference objects."""

import os
import re
import types

import numpy as np
import pytest
import torch

from _golden import load

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a B200")]


def _binding_namespace():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = next(b for b in re.findall(r"```python\n(.*?)```", text, flags=re.S) if "coo_to_csr_gee" in b)
    os.environ["LIBGEE"] = os.path.join(ROOT, "paper_2406_03726_b200", "libgee.so")
    ns = {}
    exec(compile(block, "INTEGRATION.md", "exec"), ns)
    return ns


def test_integration_binding_matches_reference_fixtures():
    from oracle import oracle as O
    ns = _binding_namespace()
    coo_to_csr_gee = ns["coo_to_csr_gee"]
    for case in load()[:40]:
        n = case["n"]
        r, c, v = O.symmetrize(case["rows"], case["cols"], case["w"], case["directed"])
        ip, cc, vv = coo_to_csr_gee(r, c, v, n, n)
        assert np.array_equal(ip, case["csr_indptr"]) and np.array_equal(cc, case["csr_cols"])
        assert np.array_equal(vv, case["csr_vals"])


def test_encode_accepts_reference_style_objects():
    """Duck-typed EdgeList / LabelVector / EmbedOptions (the reference's field names)."""
    import paper_2406_03726_b200 as G
    from oracle import oracle as O
    rng = np.random.default_rng(5)
    n, m, k = 400, 3000, 4
    rows, cols = rng.integers(0, n, m), rng.integers(0, n, m)
    w = 1.0 - rng.random(m)
    y = rng.integers(-1, k, n)
    edges = types.SimpleNamespace(n_nodes=n, rows=rows, cols=cols, weights=w, directed=False)
    labels = types.SimpleNamespace(labels=y, k_classes=k)
    opts = types.SimpleNamespace(laplacian=True, diagonal=True, correlation=True)
    z = G.encode(edges, labels, opts)
    st, zr, _ = O.encode_edges(rows, cols, w, n, False, y, k, 7)
    rown = np.sqrt((zr * zr).sum(axis=1, keepdims=True))
    assert (np.abs(z - zr) <= 1e-12 * np.maximum(np.abs(zr), rown) + 1e-15).all()
    csr = types.SimpleNamespace(n_rows=n, n_cols=n, **dict(zip(
        ("index_pointers", "col_indices", "data"), O.to_csr(rows, cols, w, n, False))))
    z2 = G.encode(csr, labels, opts)
    assert (np.abs(z2 - zr) <= 1e-12 * np.maximum(np.abs(zr), rown) + 1e-15).all()
