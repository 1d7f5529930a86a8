"""The bucketed stream encode (csrc/k_stream.cu) against the CPU oracle.

The stream path builds no CSR: it serves encode(EdgeList) for unit-weight
graphs and for weights the EdgeList found non-negative (GEE_NONNEG).  Its
sums run in any order, so Z is held to the north_star's 1e-12 (fp64) and
1e-5 (fp32 output) bars, entrywise relative to max(|z_ref|, ||z_ref row||),
with the numerically-zero-row rule of tests/test_gpu_parity.z_close.
"""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a B200")]

import paper_2406_03726_b200 as G  # noqa: E402
from paper_2406_03726_b200 import _lib  # noqa: E402
from test_gpu_parity import z_close  # noqa: E402

COMBOS = [(a, b, c) for a in (0, 1) for b in (0, 1) for c in (0, 1)]


class stream_mode:
    def __init__(self, mode):
        self.mode = mode

    def __enter__(self):
        self.old = _lib.load().gee_debug_set(_lib.DEBUG_STREAM, self.mode)

    def __exit__(self, *exc):
        _lib.load().gee_debug_set(_lib.DEBUG_STREAM, self.old)


def _launched(name):
    return name in _kernel_names()


def _kernel_names():
    lib = _lib.load()
    import ctypes
    cap = 64
    ms = (ctypes.c_float * cap)()
    nm = (ctypes.c_char_p * cap)()
    got = lib.gee_profile_read(ms, nm, cap)
    return {nm[i].decode() for i in range(max(got, 0))}


def _oracle_z(n, rows, cols, w, labels, k, directed, combo):
    f = O.flags_of(*map(bool, combo))
    st, z, _ = O.encode_edges(rows, cols, np.asarray(w, np.float64), n, directed, labels, k, f)
    return st, z


def _check(n, rows, cols, w, labels, k, directed, combos=COMBOS, dtype=torch.float64, expect_stream=True):
    edges = G.EdgeList(n, rows, cols, w, directed)
    lab = G.LabelVector(labels, k)
    for combo in combos:
        opts = G.EmbedOptions(*map(bool, combo))
        st, zr = _oracle_z(n, rows, cols, w, labels, k, directed, combo)
        if st != O.OK:
            with pytest.raises(G.NumericalDomainError):
                G.encode(edges, lab, opts, dtype=dtype)
            continue
        lib = _lib.load()
        # unit-weight graphs of <= 16384 nodes and K <= 8 default to the bitmap
        # path: switch it off so the stream path is the one under test
        old = lib.gee_debug_set(_lib.DEBUG_FORCE_BUCKETS, 2 if expect_stream else 0)
        try:
            lib.gee_profile_start(torch.cuda.current_stream().cuda_stream)
            z = G.encode(edges, lab, opts, dtype=dtype)
            lib.gee_profile_stop()
        finally:
            lib.gee_debug_set(_lib.DEBUG_FORCE_BUCKETS, old)
        names = _kernel_names()
        if expect_stream:
            assert "k_st_embed" in names, names
        pre = None
        if combo[2]:
            _, pre = _oracle_z(n, rows, cols, w, labels, k, directed, (combo[0], combo[1], 0))
        if dtype == torch.float32:
            assert z.dtype == np.float32
            z_close(z.astype(np.float64), zr, rtol=1e-5, zr_pre=pre)
        else:
            z_close(z, zr, zr_pre=pre)


def _graph(rng, n, m, wkind, loops=True, dups=True):
    rows = rng.integers(0, n, m)
    cols = rng.integers(0, n, m)
    if not loops:
        keep = rows != cols
        rows, cols = rows[keep], cols[keep]
    if dups and rows.size > 4:
        j = rng.integers(0, rows.size, rows.size // 4)
        rows = np.concatenate([rows, rows[j]])
        cols = np.concatenate([cols, cols[j]])
    m = rows.size
    if wkind == "unit":
        w = np.ones(m)
    elif wkind == "f64":
        w = 1.0 - rng.random(m)
    elif wkind == "f32":
        w = (1.0 - rng.random(m)).astype(np.float32)
    elif wkind == "zeros":
        w = np.where(rng.random(m) < 0.3, 0.0, rng.random(m))
    else:  # dyadic: exact sums in any order
        w = rng.integers(0, 8, m) / 8.0
    return rows.astype(np.int64), cols.astype(np.int64), w


@pytest.mark.parametrize("seed", range(12))
def test_stream_fuzz(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.choice([2, 3, 17, 300, 4097, 20000]))
    k = int(rng.choice([1, 2, 3, 9, 20, 50, 130]))
    m = int(rng.integers(1, 6 * n + 2))
    wkind = ["unit", "f64", "f32", "zeros", "dyadic"][seed % 5]
    directed = bool(seed % 2)
    rows, cols, w = _graph(rng, n, m, wkind)
    labels = rng.integers(-1, k, n)
    _check(n, rows, cols, w, labels, k, directed)


@pytest.mark.parametrize("k", [3, 50, 1000])
def test_stream_split_buckets(k):
    """A hub row and a dense bucket: items split, partial tiles reduce through
    the scratch tiles and the last item runs the epilogue."""
    rng = np.random.default_rng(k)
    n, m = 40000, 300000
    rows = rng.integers(0, n, m)
    rows[:120000] = 7          # hub row: one bucket holds > C entries
    rows[120000:180000] = rng.integers(0, 64, 60000)
    cols = rng.integers(0, n, m)
    w = 1.0 - rng.random(m)
    labels = rng.integers(-1, k, n)
    _check(n, rows.astype(np.int64), cols.astype(np.int64), w, labels, k, False,
           combos=[(1, 1, 1), (0, 0, 0), (1, 0, 1)])
    _check(n, rows.astype(np.int64), cols.astype(np.int64), np.ones(m), labels, k, True,
           combos=[(1, 1, 1)])


def test_stream_empty_rows_and_unlabeled():
    rng = np.random.default_rng(5)
    n = 70000
    rows = rng.integers(0, 50, 2000)  # most rows (and buckets) empty
    cols = rng.integers(0, n, 2000)
    labels = rng.integers(-1, 4, n)
    labels[:10] = -1
    _check(n, rows, cols, np.ones(2000), labels, 4, False)


@pytest.mark.timeout(600, method="thread")
def test_stream_runs_of_empty_items():
    """Runs of empty buckets between non-empty ones: a CTA passes empty work
    items without calling its stage cursor, which must not fall behind the
    descriptor ring (the R-MAT tail of configs[3] hung the embed in ~40% of
    bench runs before the cursor restarted at the current item).  Repeated
    encodes, each against the oracle."""
    rng = np.random.default_rng(11)
    n, k = 1 << 21, 50  # 64-row buckets: 32768 buckets
    bands = np.arange(0, n, 64 * 37)  # one populated bucket in 37
    rows = np.concatenate([rng.integers(0, 4096, 300000),  # a dense head (many stages)
                           (bands[rng.integers(0, bands.size, 200000)] + rng.integers(0, 64, 200000))])
    cols = rng.integers(0, n, rows.size)
    w = (1.0 - rng.random(rows.size)).astype(np.float32)
    labels = rng.integers(0, k, n)
    combo = (1, 1, 1)
    st, zr = _oracle_z(n, rows, cols, w, labels, k, True, combo)
    assert st == O.OK
    _, pre = _oracle_z(n, rows, cols, w, labels, k, True, (1, 1, 0))
    edges = G.EdgeList(n, rows.astype(np.int64), cols.astype(np.int64), w, True)
    lab = G.LabelVector(labels, k)
    for _ in range(12):
        z = G.encode(edges, lab, G.EmbedOptions(True, True, True))
        z_close(z, zr, zr_pre=pre)


@pytest.mark.parametrize("idx,scale_down", [(2, 3), (3, 5), (4, 4)])
def test_stream_configs_reduced(idx, scale_down):
    from oracle import gen
    c = gen.host_config(idx, scale_down)
    f = c["flags"]
    combo = (int(bool(f & 1)), int(bool(f & 2)), int(bool(f & 4)))
    _check(c["n"], c["rows"], c["cols"], c["weights"], c["labels"], c["k"], c["directed"], combos=[combo])


@pytest.mark.parametrize("seed", range(4))
def test_stream_fp32(seed):
    rng = np.random.default_rng(77 + seed)
    n, k = int(rng.choice([500, 30000])), int(rng.choice([3, 50, 1000]))
    rows, cols, w = _graph(rng, n, 8 * n, ["unit", "f64", "f32", "zeros"][seed])
    labels = rng.integers(-1, k, n)
    _check(n, rows, cols, w, labels, k, bool(seed % 2), combos=[(1, 1, 1), (0, 0, 0), (1, 0, 0)],
           dtype=torch.float32)


def test_fp32_signed_weights_narrowed():
    """float32 Z of a signed-weight graph: the exact f64 path, narrowed once."""
    rng = np.random.default_rng(3)
    n, k = 800, 5
    rows, cols, _ = _graph(rng, n, 6000, "unit")
    w = rng.random(rows.size) - 0.4
    labels = rng.integers(0, k, n)
    _check(n, rows, cols, w, labels, k, False, combos=[(0, 1, 1), (0, 0, 0)], dtype=torch.float32,
           expect_stream=False)


def test_signed_weights_take_exact_path():
    rng = np.random.default_rng(4)
    n, k = 600, 4
    rows, cols, _ = _graph(rng, n, 5000, "unit")
    w = rng.random(rows.size) - 0.3
    labels = rng.integers(0, k, n)
    edges = G.EdgeList(n, rows, cols, w)
    assert edges.nonneg is False
    _check(n, rows, cols, w, labels, k, False, combos=[(1, 1, 1), (0, 1, 0)], expect_stream=False)


def test_false_nonneg_assertion_recovers():
    """GEE_NONNEG asserted on a signed list: the device flags it and the
    plan recomputes on the exact path."""
    rng = np.random.default_rng(9)
    n, k = 3000, 6
    rows, cols, _ = _graph(rng, n, 20000, "unit")
    w = rng.random(rows.size) - 0.2
    labels = rng.integers(0, k, n)
    dev = torch.device("cuda")
    r, c, wt, lab = (torch.as_tensor(x, device=dev) for x in (rows, cols, w, labels))
    enc = G.GeeEncoder(n, rows.size, k, False, G.EmbedOptions(True, True, True), dev, nonneg=True)
    enc.err.zero_()
    enc.run(r, c, wt, lab, check=False)
    assert int(enc.err.item()) & _lib.ERR_NEG_WEIGHT
    z = enc.run(r, c, wt, lab, check=True).cpu().numpy()
    st, zr = _oracle_z(n, rows, cols, w, labels, k, False, (1, 1, 1))
    assert st == O.OK
    _, pre = _oracle_z(n, rows, cols, w, labels, k, False, (1, 1, 0))
    z_close(z, zr, zr_pre=pre)


def test_stream_range_errors():
    n = 5000
    rows = np.arange(100) % n
    cols = np.arange(100) % n
    cols[50] = n + 3
    edges = G.EdgeList(n, rows, cols, None, validate=False)  # unit weights: the stream path
    with pytest.raises(G.StructuralError):
        G.encode(edges, G.LabelVector(np.zeros(n, np.int64), 2), G.EmbedOptions(True, False, True))


def test_stream_matches_csr_path():
    """Stream and exact CSR paths agree (both within 1e-12 of the oracle)."""
    rng = np.random.default_rng(12)
    n, k = 50000, 20
    rows, cols, w = _graph(rng, n, 400000, "f64")
    labels = rng.integers(-1, k, n)
    edges = G.EdgeList(n, rows, cols, w)
    lab = G.LabelVector(labels, k)
    opts = G.EmbedOptions(True, True, True)
    z1 = G.encode(edges, lab, opts)
    with stream_mode(1):
        z2 = G.encode(edges, lab, opts)
    rown = np.sqrt((z2 * z2).sum(axis=1, keepdims=True))
    assert (np.abs(z1 - z2) <= 2e-12 * np.maximum(np.abs(z2), rown) + 1e-14).all()


def test_stream_all_ones_key():
    """N = 2^23 with K <= 8: 512-row buckets and 23 column bits would make the
    entry (row % 512 == 511, col == N - 1) the 32-bit key 0xffffffff, which is
    the embed's "no entry" marker.  The geometry keeps row-in-bucket + column
    within 31 bits, so the entry counts (it was dropped before)."""
    n, k = 1 << 23, 4
    rng = np.random.default_rng(5)
    rows = np.concatenate([np.array([511, 1023, n - 1, 511]), rng.integers(0, n, 5000)]).astype(np.int64)
    cols = np.concatenate([np.array([n - 1, n - 1, n - 1, 7]), rng.integers(0, n, 5000)]).astype(np.int64)
    w = 1.0 - rng.random(rows.size)
    labels = rng.integers(0, k, n)
    _check(n, rows, cols, w, labels, k, True, combos=[(0, 0, 0), (1, 1, 1)])
