"""On-device generators (csrc/k_gen.cu) against their C
restatement (oracle/gee_gen.c): the two arms must draw the SAME graph, so
the comparison is bit-exact on every array."""

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a B200")]


def _np(x):
    return x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


@pytest.mark.parametrize("idx,scale_down", [(0, 0), (2, 3), (2, 0), (3, 6), (3, 2), (4, 4)])
def test_device_generator_equals_host(idx, scale_down):
    from oracle import gen
    from paper_2406_03726_b200 import synth
    d = synth.make_config(idx, "cuda", scale_down)
    h = gen.host_config(idx, scale_down)
    assert d["n"] == h["n"] and d["e"] == h["e"] and d["k"] == h["k"]
    for key in ("rows", "cols", "weights", "labels"):
        a, b = _np(d[key]), _np(h[key])
        assert a.dtype == b.dtype, key
        assert np.array_equal(a, b), f"{key} differs at config {idx} (scale_down {scale_down})"


def test_gnm_first_occurrence_rule():
    """Candidates repeating an earlier pair are skipped in candidate order."""
    from oracle import gen
    from paper_2406_03726_b200 import _device, _lib, synth
    n, count = 50, 4000  # tiny n: many repeats
    key = synth.stream_key(11, synth.S_PAIRS)
    keys = torch.empty(count, dtype=torch.int64, device="cuda")
    _lib.check(_lib.load().gee_gen_pairs(key, 0, count, n, _device.ptr(keys), _device.stream_handle()))
    ref = gen.pairs(key, 0, count, n)
    assert np.array_equal(keys.cpu().numpy(), ref)
    seen, first = set(), []
    for k in ref.tolist():
        if k >= 0 and k not in seen:
            seen.add(k)
            first.append(k)
    m = len(first)
    rows = np.empty(m, np.int64)
    cols = np.empty(m, np.int64)
    assert gen._lib().ggen_gnm(key, n, m, count, rows.ctypes.data, cols.ctypes.data) > 0
    assert np.array_equal(rows * n + cols, np.array(first))
