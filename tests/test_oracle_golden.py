"""Pin the CPU oracle (oracle/gee_oracle.c) to the reference's own outputs.

Every array the reference produced for the committed fixtures must be
reproduced BITWISE (np.array_equal + dtype), including errors.
"""

import numpy as np
import pytest

from _golden import COMBOS, load, ztag
from oracle import oracle as O

CASES = load()


def _eq(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return a.dtype == b.dtype and a.shape == b.shape and np.array_equal(a, b)


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_matches_reference_bitwise(case):
    n, k, directed = case["n"], case["k"], case["directed"]
    ip, oc, ov = O.to_csr(case["rows"], case["cols"], case["w"], n, directed)
    assert _eq(ip, case["csr_indptr"]) and _eq(oc, case["csr_cols"]) and _eq(ov, case["csr_vals"])
    aug = O.add_identity(ip, oc, ov, n)
    assert _eq(aug[0], case["aug_indptr"]) and _eq(aug[1], case["aug_cols"])
    assert _eq(aug[2], case["aug_vals"])
    # np.bincount returns int64 zeros when the CSR is empty (sparse.py:196);
    # values are what degrees mean, so compare them as float64
    assert _eq(O.degree(ip, ov, n), case["deg"].astype(np.float64))
    assert _eq(O.degree(aug[0], aug[2], n), case["deg_aug"].astype(np.float64))
    lap = O.laplacian_normalize(ip, oc, ov, n, case["deg"])
    if "lap_error" in case:
        assert lap is None
    else:
        assert _eq(lap[0], case["lap_indptr"]) and _eq(lap[1], case["lap_cols"])
        assert _eq(lap[2], case["lap_vals"])
    assert _eq(O.class_counts(case["labels"], k), case["counts"])
    for lap_f, diag_f, corr_f in COMBOS:
        tag = ztag(lap_f, diag_f, corr_f)
        st, z, _ = O.encode_edges(case["rows"], case["cols"], case["w"], n, directed,
                                  case["labels"], k, O.flags_of(lap_f, diag_f, corr_f))
        if tag + "_error" in case:
            assert st != O.OK
        else:
            assert st == O.OK
            assert _eq(z, case[tag]), (tag, np.abs(z - case[tag]).max())


def test_fixture_covers_edge_cases():
    names = {c["name"] for c in CASES}
    assert {"triangle", "edgeless", "all_unlabeled", "cancel_dup", "neg_degree",
            "triple_dup"} <= names
    assert any(c["directed"] for c in CASES) and any(not c["directed"] for c in CASES)
    assert any("z101_error" in c or "z100_error" in c for c in CASES)


def test_triangle_hand_goldens():
    # test_embedding.py:48-63
    rows, cols, w, lab = [0, 0, 1], [1, 2, 2], [1.0, 1.0, 1.0], [0, 1, 1]
    st, z, _ = O.encode_edges(rows, cols, w, 3, False, lab, 2, 0)
    assert np.allclose(z, [[0.0, 1.0], [1.0, 0.5], [1.0, 0.5]], atol=1e-15)
    st, z, _ = O.encode_edges(rows, cols, w, 3, False, lab, 2, O.DIAGONAL)
    assert np.allclose(z, np.ones((3, 2)), atol=1e-15)
    st, z, _ = O.encode_edges(rows, cols, w, 3, False, lab, 2, O.LAPLACIAN)
    assert np.allclose(z, [[0.0, 0.5], [0.5, 0.25], [0.5, 0.25]], atol=1e-15)


def test_correlate_goldens():
    # test_embedding.py:81-98
    assert np.array_equal(O.correlate_rows(np.array([[3.0, 4.0]])), [[0.6, 0.8]])
    assert np.array_equal(O.correlate_rows(np.array([[0.0, 0.0]])), [[0.0, 0.0]])
    assert np.array_equal(O.correlate_rows(np.array([[0.0, 7.0]])), [[0.0, 1.0]])
    assert O.correlate_rows(np.array([[np.nan, 1.0]])) is None


def test_csr_fig1_walkthrough():
    # test_sparse.py:30-43 / PAPER.md Fig. 1
    ip, oc, ov = O.coo_to_csr([0, 0, 1, 2, 2], [0, 3, 2, 1, 5], [1.0, 1.0, 1.0, 2.0, 3.0], 3, 6)
    assert ip[2] == 3 and ip[3] == 5
    assert oc[3:5].tolist() == [1, 5] and ov[3:5].tolist() == [2.0, 3.0]
