"""Host-side logic that runs without a GPU: container validation mirrors the
reference, generators are seeded and shaped as BASELINE.json says, and the
product path refuses to run without the device (no CPU fallback)."""

import numpy as np
import pytest
import torch

from paper_2406_03726_b200 import (EdgeList, EmbedOptions, GpuUnavailableError, LabelVector,
                                   StructuralError, encode, synth)


def test_edgelist_validation_matches_reference_rules():
    with pytest.raises(StructuralError, match="equal length"):
        EdgeList(3, [0, 1], [1], [1.0, 1.0])
    with pytest.raises(StructuralError, match="outside node range"):
        EdgeList(3, [0, 3], [1, 1], [1.0, 1.0])
    with pytest.raises(StructuralError, match="outside node range"):
        EdgeList(3, [0, -1], [1, 1], [1.0, 1.0])
    with pytest.raises(StructuralError, match="finite"):
        EdgeList(3, [0, 1], [1, 2], [1.0, np.inf])
    e = EdgeList(3, [0, 1], [1, 2], np.array([1.0, 2.0], np.float32))
    assert e.weights.dtype == np.float32 and e.n_edges == 2
    assert e.weights_f64().dtype == np.float64
    assert EdgeList(4).n_edges == 0


def test_labelvector_validation_matches_reference_rules():
    with pytest.raises(StructuralError):
        LabelVector(np.array([0]), 0)
    with pytest.raises(StructuralError):
        LabelVector(np.array([0, -2]), 2)
    with pytest.raises(StructuralError, match="exceeds"):
        LabelVector(np.array([0, 2]), 2)
    assert LabelVector.from_values([0, 3, -1]).k_classes == 4
    with pytest.raises(StructuralError):
        LabelVector.from_values([-1, -1])


def test_embed_options():
    combos = EmbedOptions.all_combinations()
    assert len(combos) == 8 and len({c.flags for c in combos}) == 8
    assert EmbedOptions(True, True, True).flags == 7


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    e = EdgeList(3, [0, 0, 1], [1, 2, 2], [1.0, 1.0, 1.0])
    with pytest.raises(GpuUnavailableError):
        encode(e, LabelVector(np.array([0, 1, 1]), 2))
    with pytest.raises(GpuUnavailableError):
        e.to_csr()


def test_zipf_counts():
    c = synth.zipf_counts(1_000_000, 1000, 1.5)
    assert c.sum() == 1_000_000 and c[0] == c.max()
    assert abs(c[0] / 1e6 - 0.3924) < 0.01
    c20 = synth.zipf_counts(600_000, 20, 1.1)
    assert c20.sum() == 600_000 and c20.min() > 6000


def test_sbm_config_shape_and_determinism():
    from oracle import gen
    a = gen.host_config(0)
    b = gen.host_config(1)
    assert np.array_equal(a["rows"], b["rows"]) and np.array_equal(a["cols"], b["cols"])
    assert a["n"] == 10_000 and a["k"] == 3 and not a["directed"]
    assert 5_400_000 < a["e"] < 5_600_000
    assert (a["rows"] < a["cols"]).all()  # i < j, no self loops, no duplicates
    assert b["flags"] == 7 and a["flags"] == 0
    # row-major order, like the reference's pair sweep
    key = a["rows"] * a["n"] + a["cols"]
    assert (np.diff(key) > 0).all()


def test_scaled_generators():
    from oracle import gen
    c2 = gen.host_config(2, scale_down=6)
    assert c2["weights"].dtype == np.float64 and (c2["weights"] > 0).all() and (c2["weights"] <= 1).all()
    assert np.bincount(c2["labels"]).tolist() == synth.zipf_counts(c2["n"], 20, 1.1).tolist()
    c3 = gen.host_config(3, scale_down=8)
    assert c3["directed"] and c3["weights"].dtype == np.float32 and c3["n"] == 1 << 16
    assert int(c3["rows"].max()) < c3["n"] and int(c3["cols"].max()) < c3["n"]
    assert (c3["weights"] > 0).all() and (c3["weights"] <= 1).all()
    # R-MAT skew: P(row bit = 1) = c + d = 0.24 per level
    assert abs((c3["rows"] & 1).mean() - 0.24) < 0.01 and abs((c3["cols"] & 1).mean() - 0.24) < 0.01
    c4 = gen.host_config(4, scale_down=8)
    keys = c4["rows"] * c4["n"] + c4["cols"]
    assert np.unique(keys).size == keys.size and bool((c4["rows"] < c4["cols"]).all())


def test_generator_is_counter_based():
    """Edge i depends only on (seed, i): a prefix of a longer draw is the
    shorter draw, and python's key derivation equals the C one."""
    from oracle import gen
    assert gen._lib().ggen_key(3, synth.S_RMAT) == synth.stream_key(3, synth.S_RMAT)
    a = gen.pairs(synth.stream_key(4, synth.S_PAIRS), 0, 5000, 1000)
    b = gen.pairs(synth.stream_key(4, synth.S_PAIRS), 1000, 4000, 1000)
    assert np.array_equal(a[1000:], b)
    labs = synth.uniform_labels(9, 100000, 7)
    assert set(np.unique(labs)) == set(range(7)) and abs(np.bincount(labs).std() / 100000 * 7) < 0.02
