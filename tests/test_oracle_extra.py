"""Pin tests/golden/reference_extra.npz (made from the reference by
tests/golden/make_extra_golden.py) against the CPU oracle: W and the
from_triplets CSRs bitwise, encode_reference within the reference's own
pipeline-agreement tolerance of the oracle's encode (cli.py:40, 1e-12)."""

import numpy as np
import pytest

from _golden import COMBOS, load_extra, rtag
from oracle import oracle as O

CASES = load_extra()


def _eq(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.dtype == b.dtype and a.shape == b.shape and np.array_equal(a, b)


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_extra_fixtures_match_oracle(case):
    n, k, directed = case["n"], case["k"], case["directed"]
    ip, c, v = O.weight_matrix(case["labels"], k)
    assert _eq(ip, case["wm_indptr"]) and _eq(c, case["wm_cols"]) and _eq(v, case["wm_vals"])
    for tag, nc in (("ft", n), ("ftr", n + 3)):
        ip, c, v = O.coo_to_csr(case["rows"], case["cols"], case["w"], n, nc)
        assert _eq(ip, case[tag + "_indptr"]) and _eq(c, case[tag + "_cols"]) and _eq(v, case[tag + "_vals"])
    for lap, diag, corr in COMBOS:
        tag = rtag(lap, diag, corr)
        st, z, _ = O.encode_edges(case["rows"], case["cols"], case["w"], n, directed, case["labels"], k,
                                  O.flags_of(bool(lap), bool(diag), bool(corr)))
        if tag + "_error" in case:
            assert str(case[tag + "_error"]) == "NumericalDomainError" and st == O.E_NEG_DEGREE
            continue
        assert st == O.OK
        zr = case[tag]
        if corr:  # numerically-zero rows are normalised differently by the two pipelines
            zp = case[rtag(lap, diag, 0)]
            live = np.sqrt((zp * zp).sum(axis=1)) > 1e-12 * max(1.0, float(np.abs(zp).max())) if zp.size else []
            z, zr = z[live], zr[live]
        rown = np.sqrt((zr * zr).sum(axis=1, keepdims=True)) if zr.size else zr
        assert (np.abs(z - zr) <= np.maximum(1e-12 * np.maximum(np.abs(zr), rown), 1e-14)).all(), case["name"]
