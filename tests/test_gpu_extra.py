"""GPU parity of the remaining reference entry points against fixtures made by
the reference itself (tests/golden/reference_extra.npz):

* build_weight_matrix   (embedding.py:92-107)  -- gee_weight_matrix, bitwise
* CsrMatrix.from_triplets (sparse.py:33-68)    -- gee_csr_build, bitwise,
  square and rectangular, numpy and device inputs, and its range / finiteness
  errors for device inputs
* encode_reference      (embedding.py:146-200) -- within 1e-12 of the
  reference's encode_reference, our EdgeList and a duck-typed one
"""

import os
import sys
from types import SimpleNamespace

import numpy as np
import pytest
import torch

from _golden import COMBOS, load_extra, rtag

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a B200")]

import paper_2406_03726_b200 as G  # noqa: E402
from test_gpu_parity import csr_equal, same, z_close  # noqa: E402

CASES = load_extra()


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_build_weight_matrix_bitwise(case):
    w = G.build_weight_matrix(G.LabelVector(case["labels"], case["k"]))
    assert (w.n_rows, w.n_cols) == (case["n"], case["k"])
    assert csr_equal(w, (case["wm_indptr"], case["wm_cols"], case["wm_vals"]))


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_from_triplets_bitwise(case):
    n = case["n"]
    for tag, nc in (("ft", n), ("ftr", n + 3)):
        ref = (case[tag + "_indptr"], case[tag + "_cols"], case[tag + "_vals"])
        m = G.CsrMatrix.from_triplets(case["rows"], case["cols"], case["w"], n, nc)
        assert csr_equal(m, ref)
        d = lambda a, t: torch.as_tensor(np.asarray(a), dtype=t, device="cuda")  # noqa: E731
        m = G.CsrMatrix.from_triplets(d(case["rows"], torch.int64), d(case["cols"], torch.int64),
                                      d(case["w"], torch.float64), n, nc)
        assert csr_equal(m, ref)


def test_from_triplets_device_input_errors():
    d = lambda a, t: torch.tensor(a, dtype=t, device="cuda")  # noqa: E731
    with pytest.raises(G.StructuralError, match="outside"):
        G.CsrMatrix.from_triplets(d([0, 3], torch.int64), d([1, 0], torch.int64), d([1.0, 1.0], torch.float64), 3, 3)
    with pytest.raises(G.StructuralError, match="outside"):
        G.CsrMatrix.from_triplets(d([0, -1], torch.int64), d([1, 0], torch.int64), d([1.0, 1.0], torch.float64), 3, 3)
    with pytest.raises(G.StructuralError, match="finite"):
        G.CsrMatrix.from_triplets(d([0, 1], torch.int64), d([1, 0], torch.int64),
                                  d([1.0, float("nan")], torch.float64), 3, 3)


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_encode_reference_matches_reference(case):
    n, k, directed = case["n"], case["k"], case["directed"]
    labels = G.LabelVector(case["labels"], k)
    ours = G.EdgeList(n, case["rows"], case["cols"], case["w"], directed)
    duck = SimpleNamespace(n_nodes=n, rows=np.asarray(case["rows"]), cols=np.asarray(case["cols"]),
                           weights=np.asarray(case["w"], np.float64), directed=directed)
    for lap, diag, corr in COMBOS:
        opts = G.EmbedOptions(bool(lap), bool(diag), bool(corr))
        tag = rtag(lap, diag, corr)
        for edges in (ours, duck):
            if tag + "_error" in case:
                with pytest.raises(getattr(G, str(case[tag + "_error"]))):
                    G.encode_reference(edges, labels, opts)
            else:
                pre = case[rtag(lap, diag, 0)] if corr else None
                z_close(G.encode_reference(edges, labels, opts), case[tag], zr_pre=pre)


def test_encode_reference_checks_only_label_count():
    e = G.EdgeList(3, [0, 0, 1], [1, 2, 2], [1.0, 1.0, 1.0])
    with pytest.raises(G.StructuralError, match="label count"):
        G.encode_reference(e, G.LabelVector(np.array([0, 1]), 2))


def test_encode_reference_overflow_is_not_an_error():
    # finite weights whose sums overflow: encode raises (embedding.py:137-138),
    # encode_reference divides by the inf norm as numpy does (embedding.py:195-199)
    e = G.EdgeList(2, [0, 0], [1, 1], [1.5e308, 1.5e308], directed=True)
    lab = G.LabelVector(np.array([-1, 0]), 1)  # n_0 = 1: z[0, 0] = 1.5e308 + 1.5e308 = inf
    opts = G.EmbedOptions(correlation=True)
    with pytest.raises(G.NumericalDomainError):
        G.encode(e, lab, opts)
    with np.errstate(all="ignore"):
        ref = np.array([[np.inf], [0.0]])
        norms = np.sqrt((ref * ref).sum(axis=1))
        ref[norms > 0] /= norms[norms > 0, None]
    z = G.encode_reference(e, lab, opts)
    assert np.array_equal(np.isnan(z), np.isnan(ref)) and same(np.nan_to_num(z), np.nan_to_num(ref))


def test_bench_cli_reference_pipelines(tmp_path, capsys):
    from paper_2406_03726_b200 import bench_cli
    rng = np.random.default_rng(3)
    n = 300
    r, c = np.nonzero(np.triu(rng.random((n, n)) < 0.05, 1))
    w = 1.0 - rng.random(r.size)
    e = tmp_path / "g.txt"
    e.write_text("".join(f"{i} {j} {float(x)!r}\n" for i, j, x in zip(r, c, w)))
    lab = tmp_path / "y.txt"
    lab.write_text("".join(f"{x}\n" for x in rng.integers(0, 3, n)))
    for p in ("sparse", "reference", "gpu", "gpu-ops"):
        assert bench_cli.main(["bench", "--edges", str(e), "--labels", str(lab), "--all-options",
                               "--pipeline", p, "--repeats", "1"]) == 0
    out = capsys.readouterr().out
    assert out.count("dataset,pipeline") == 4
