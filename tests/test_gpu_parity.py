"""GPU parity: every device op against the reference's own outputs (committed
fixtures) and against the CPU oracle (oracle/gee_oracle.c, itself pinned
bitwise to the reference).

Bars (north_star): n_k, CSR structure+values, degrees and the materialised
A+I / Laplacian CSRs BIT-EXACT; Z within relative 1e-12 in fp64, measured as
|dz| <= 1e-12 * max(|z_ref|, ||z_ref row||_2) entrywise (SURVEY Appendix A:
entrywise-relative for non-negative weights, row-relative when signed
weights can cancel).
"""

import numpy as np
import pytest
import torch

from _golden import COMBOS, load, ztag
from oracle import oracle as O

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a B200")]

import paper_2406_03726_b200 as G  # noqa: E402

RTOL = 1e-12
CASES = load()
PATHS = ["default", "sort", "buckets", "sort64"]


class assembly_path:
    """Select the CSR-assembly path via the library's test hook: "default"
    (column bitmaps for unit-weight graphs with <= 16384 nodes, else the
    radix sort when (row, col) packs into 32 bits or the graph is weighted,
    else row buckets),
    "sort" (never the bitmap path), "buckets" (always row buckets) or
    "sort64" (the radix sort also on 64-bit (row, col) keys)."""

    def __init__(self, path):
        self.force = {"default": 0, "sort": 2, "buckets": 1, "sort64": 3}[path]

    def __enter__(self):
        # a forced CSR path also disables the bucketed stream encode, so
        # encode(EdgeList) runs through the CSR assembly under test
        from paper_2406_03726_b200 import _lib
        self.old = _lib.load().gee_debug_set(_lib.DEBUG_FORCE_BUCKETS, self.force)
        self.old_stream = _lib.load().gee_debug_set(_lib.DEBUG_STREAM, 1 if self.force else 0)

    def __exit__(self, *exc):
        from paper_2406_03726_b200 import _lib
        _lib.load().gee_debug_set(_lib.DEBUG_FORCE_BUCKETS, self.old)
        _lib.load().gee_debug_set(_lib.DEBUG_STREAM, self.old_stream)


def z_close(z, zr, rtol=RTOL, zr_pre=None):
    """Compare Z with the reference.  `zr_pre` is the reference's Z before
    correlation: a row whose terms cancel to within rounding (norm below
    1e-12 of the matrix scale) is numerically zero -- the reference's left
    fold leaves exactly 0.0 or some ~1e-17 there, any other order leaves a
    different ~1e-17, and correlate_rows scales that to a unit row (the
    reference's own encode_reference disagrees with encode the same way,
    e.g. fixture triple_dup).  Those rows are compared before normalisation
    (the same combo without correlation is checked too) and skipped after."""
    z = np.asarray(z)
    zr = np.asarray(zr)
    assert z.shape == zr.shape and z.dtype == np.float64
    if zr_pre is not None and zr.size:
        zp = np.asarray(zr_pre)
        scale = max(1.0, float(np.abs(zp).max()))
        live = np.sqrt((zp * zp).sum(axis=1)) > 1e-12 * scale
        z, zr = z[live], zr[live]
    rown = np.sqrt((zr * zr).sum(axis=1, keepdims=True)) if zr.size else zr
    # signed weights can cancel a whole row to ~0 (the reference then holds an
    # exact 0.0 where any other summation order leaves ~1e-17): a 1e-14
    # absolute floor, 100x tighter than the reference's own 1e-12 absolute
    # oracle test (test_embedding.py:130)
    bound = np.maximum(rtol * np.maximum(np.abs(zr), rown), 1e-14)
    bad = np.abs(z - zr) > bound
    assert not bad.any(), f"max |dz|={np.abs(z - zr).max():.3e} at {np.argwhere(bad)[:3]}"


def same(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return a.shape == b.shape and np.array_equal(a, b)


def csr_equal(m, ref):
    ip, c, v = m.to_numpy()
    return same(ip, ref[0]) and same(c, ref[1]) and same(v, ref[2]) and v.dtype == np.float64


# ---- reference fixtures ------------------------------------------------------
@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_reference_fixture(case, path):
    with assembly_path(path):
        _reference_fixture(case)


def _reference_fixture(case):
    n, k, directed = case["n"], case["k"], case["directed"]
    edges = G.EdgeList(n, case["rows"], case["cols"], case["w"], directed)
    labels = G.LabelVector(case["labels"], k)
    csr = edges.to_csr()
    assert csr_equal(csr, (case["csr_indptr"], case["csr_cols"], case["csr_vals"]))
    csr.validate()
    aug = G.add_identity(csr)
    assert csr_equal(aug, (case["aug_indptr"], case["aug_cols"], case["aug_vals"]))
    deg = G.degree_vector(csr).cpu().numpy()
    assert same(deg, case["deg"].astype(np.float64))
    deg_aug = G.degree_vector(csr, diagonal=True).cpu().numpy()
    assert same(deg_aug, case["deg_aug"].astype(np.float64))
    assert same(G.degree_vector(aug).cpu().numpy(), case["deg_aug"].astype(np.float64))
    if "lap_error" in case:
        with pytest.raises(G.NumericalDomainError):
            G.laplacian_normalize(csr, deg)
    else:
        lap = G.laplacian_normalize(csr, deg)
        assert csr_equal(lap, (case["lap_indptr"], case["lap_cols"], case["lap_vals"]))
    assert same(labels.class_counts(), case["counts"])
    for lap_f, diag_f, corr_f in COMBOS:
        opts = G.EmbedOptions(bool(lap_f), bool(diag_f), bool(corr_f))
        tag = ztag(lap_f, diag_f, corr_f)
        for adj in (edges, csr):
            if tag + "_error" in case:
                with pytest.raises(G.NumericalDomainError):
                    G.encode(adj, labels, opts)
            else:
                pre = case[ztag(lap_f, diag_f, 0)] if corr_f else None
                z_close(G.encode(adj, labels, opts), case[tag], zr_pre=pre)


def test_triangle_goldens():
    # test_embedding.py:48-63
    e = G.EdgeList(3, [0, 0, 1], [1, 2, 2], [1.0, 1.0, 1.0])
    lab = G.LabelVector(np.array([0, 1, 1]), 2)
    assert np.allclose(G.encode(e.to_csr(), lab), [[0, 1], [1, .5], [1, .5]], atol=1e-15)
    assert np.allclose(G.encode(e, lab, G.EmbedOptions(diagonal=True)), np.ones((3, 2)), atol=1e-15)
    assert np.allclose(G.encode(e, lab, G.EmbedOptions(laplacian=True)),
                       [[0, .5], [.5, .25], [.5, .25]], atol=1e-15)
    z = G.encode(G.EdgeList(2, [0], [1], [1.0]), G.LabelVector(np.array([0, 1]), 2))
    assert np.array_equal(z, [[0.0, 1.0], [1.0, 0.0]])


def test_structural_errors():
    e = G.EdgeList(3, [0, 0, 1], [1, 2, 2], [1.0, 1.0, 1.0])
    with pytest.raises(G.StructuralError):
        G.encode(e, G.LabelVector(np.array([0, 1]), 2))
    with pytest.raises(G.StructuralError):
        G.encode(e.to_csr(), G.LabelVector(np.array([0, 1]), 2))
    rect = G.CsrMatrix.from_triplets([0], [2], [1.0], 2, 3)
    with pytest.raises(G.StructuralError, match="square"):
        G.encode(rect, G.LabelVector(np.array([0, 1]), 2))
    # device-side label validation (labels handed in as a CUDA tensor)
    bad = G.LabelVector(torch.tensor([0, 5, 1], device="cuda"), 2)
    with pytest.raises(G.StructuralError):
        G.encode(e, bad)
    # device-side edge validation
    with pytest.raises(G.StructuralError):
        G.EdgeList(3, torch.tensor([0, 7], device="cuda"), torch.tensor([1, 1], device="cuda"),
                   torch.tensor([1.0, 1.0], device="cuda", dtype=torch.float64))


# ---- oracle fuzz -------------------------------------------------------------
def _graph(rng, n, m, kind, directed, k, dup_runs=False, hub=None):
    rows = rng.integers(0, n, m)
    cols = rng.integers(0, n, m)
    if hub is not None:
        sel = rng.random(m) < hub[1]
        rows[sel] = hub[0]
    if dup_runs and m >= 40:
        for t in range(0, m - 8, 37):  # runs of 2..6 identical coordinates
            ln = 2 + (t % 5)
            rows[t:t + ln] = rows[t]
            cols[t:t + ln] = cols[t]
    if kind == "unit":
        w = np.ones(m)
    elif kind == "pos":
        w = 1.0 - rng.random(m)
    elif kind == "signed":
        w = rng.uniform(-2, 2, m)
    elif kind == "dyadic":
        w = rng.choice([-1.0, 0.5, 1.0, 2.0, 0.25], m)
    else:
        w = (1.0 - rng.random(m, dtype=np.float32)).astype(np.float32)
    labels = rng.integers(0, k, n)
    labels[rng.random(n) < 0.1] = -1
    return rows, cols, w, labels


def _check_against_oracle(n, rows, cols, w, labels, k, directed, combos=COMBOS):
    w64 = np.asarray(w, dtype=np.float64)
    edges = G.EdgeList(n, rows, cols, w, directed)
    lab = G.LabelVector(labels, k)
    ref_csr = O.to_csr(rows, cols, w64, n, directed)
    csr = edges.to_csr()
    assert csr_equal(csr, ref_csr)
    ip, oc, ov = ref_csr
    for diag in (False, True):
        if diag:
            a = O.add_identity(ip, oc, ov, n)
            dref = O.degree(a[0], a[2], n)
        else:
            dref = O.degree(ip, ov, n)
        assert same(G.degree_vector(csr, diagonal=diag).cpu().numpy(), dref)
    assert same(lab.class_counts(), O.class_counts(labels, k))
    for lap_f, diag_f, corr_f in combos:
        st, zr, ex = O.encode_edges(rows, cols, w64, n, directed, labels, k,
                                    O.flags_of(lap_f, diag_f, corr_f), want_degree=True)
        opts = G.EmbedOptions(bool(lap_f), bool(diag_f), bool(corr_f))
        if st != O.OK:
            with pytest.raises(G.NumericalDomainError):
                G.encode(edges, lab, opts)
            continue
        pre = None
        if corr_f:
            _, pre, _ = O.encode_edges(rows, cols, w64, n, directed, labels, k,
                                       O.flags_of(lap_f, diag_f, 0))
        z = G.encode(edges, lab, opts)
        z_close(z, zr, zr_pre=pre)
        z_close(G.encode(csr, lab, opts), zr, zr_pre=pre)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("seed", range(6))
def test_fuzz_small(seed, path):
    with assembly_path(path):
        _fuzz_small(seed)


def _fuzz_small(seed):
    rng = np.random.default_rng(1000 + seed)
    for kind in ("unit", "pos", "signed", "dyadic", "f32"):
        n = int(rng.integers(2, 400))
        m = int(rng.integers(0, 6 * n))
        k = int(rng.integers(1, 12))
        directed = bool(rng.integers(0, 2))
        _check_against_oracle(n, *_graph(rng, n, m, kind, directed, k, dup_runs=seed % 2 == 0),
                              k, directed)


@pytest.mark.parametrize("n,m,k,kind,directed,hub", [
    (3000, 150_000, 5, "pos", False, None),        # tier D rows (n_cols <= 12288, long rows)
    (3000, 150_000, 5, "pos", True, (17, 0.05)),   # tier D row longer than the smem stage
    (40_000, 400_000, 20, "pos", False, None),     # tiers S/B (large n)
    (40_000, 300_000, 50, "pos", True, (5, 0.1)),  # tier X hub row (LSD) + long embed row
    (20_000, 200_000, 3, "unit", False, (9, 0.2)),  # long row, register path
    (20_000, 100_000, 1000, "pos", False, (3, 0.2)),  # K=1000 shared-memory path + long row
    (5_000, 40_000, 2500, "unit", True, None),     # K > tile: tiled correlation
])
@pytest.mark.parametrize("path", PATHS)
def test_tiers(n, m, k, kind, directed, hub, path):
    rng = np.random.default_rng(n + m + k)
    with assembly_path(path):
        _check_against_oracle(n, *_graph(rng, n, m, kind, directed, k, dup_runs=True, hub=hub), k,
                          directed, combos=[(0, 0, 0), (1, 1, 1), (1, 0, 1), (0, 1, 0)])


def test_runs_of_duplicates_in_stream_order():
    # 5 identical coordinates whose sum depends on the order (non-associative)
    vals = [1e16, 1.0, -1e16, 1.0, 3.0]
    n = 20000  # large n -> tiers S/B path; repeated below with small n -> tier D
    for path in PATHS:
        for n in (20000, 50):
            rows = np.array([3] * 5 + [3] * 40, np.int64)
            cols = np.array([7] * 5 + list(range(10, 50)), np.int64)
            w = np.array(vals + [0.5] * 40)
            with assembly_path(path):
                _check_against_oracle(n, rows, cols, w, np.zeros(n, np.int64), 1, True)
                _check_against_oracle(n, cols, rows, w, np.zeros(n, np.int64), 1, False)


def test_weighted_long_rows_exact_degree_fold():
    # non-dyadic weights: the certificate fails and the sequential fold runs
    rng = np.random.default_rng(5)
    n = 30000
    rows = np.concatenate([np.full(9000, 11), rng.integers(0, n, 60000)])
    cols = rng.integers(0, n, rows.size)
    w = rng.random(rows.size) * 1e3 + 1e-9
    for path in PATHS:
        with assembly_path(path):
            _check_against_oracle(n, rows, cols, w, rng.integers(0, 4, n), 4, False,
                                  combos=[(1, 1, 1), (1, 0, 0)])


def test_large_n_multigraph_default_path():
    # n > 65535: (row, col) no longer packs into 32 bits -> 64-bit radix sort by default (weighted)
    rng = np.random.default_rng(77)
    n = 100_000
    rows = np.concatenate([np.full(6000, 4242), rng.integers(0, n, 300_000)])
    cols = rng.integers(0, n, rows.size)
    rows[:300] = 17
    cols[:300] = 23  # a 300-long duplicate run (stream-order sum)
    w = 1.0 - rng.random(rows.size)
    _check_against_oracle(n, rows, cols, w, rng.integers(-1, 7, n), 7, False,
                          combos=[(1, 1, 1), (0, 0, 0)])


def test_unit_weights_with_duplicates():
    # unit weights + duplicate coordinates: the sort path must materialise values
    rng = np.random.default_rng(3)
    n = 500
    rows = rng.integers(0, n, 20_000)
    cols = rng.integers(0, n, 20_000)
    for path in PATHS:
        with assembly_path(path):
            _check_against_oracle(n, rows, cols, np.ones(rows.size), rng.integers(0, 3, n), 3, False,
                                  combos=[(1, 1, 1), (0, 0, 0), (1, 0, 0)])


def _sorted_unit(rng, n, p):
    """Row-major (i < j) unit-weight pairs, like the SBM generator's output."""
    r, c = np.nonzero(np.triu(rng.random((n, n)) < p, 1))
    return r.astype(np.int64), c.astype(np.int64)


@pytest.mark.parametrize("variant", ["plain", "adjacent_dup", "both_directions", "loops", "directed",
                                     "max_n", "no_edges", "unlabeled", "tiny", "k1"])
def test_bitmap_encode_variants(variant):
    # the fused bitmap encode (unit weights, n <= 16384, K <= 8): warp-combined
    # atomics on sorted lists, the in-place symmetrisation, and the rare path
    # for repeated pairs (in-warp duplicate, a pair listed in both directions)
    rng = np.random.default_rng(sum(map(ord, variant)))
    n, k, directed = 3001, 5, False
    if variant == "max_n":
        n, k = 16384, 8
        rows = rng.integers(0, n, 400_000)
        cols = rng.integers(0, n, 400_000)
        o = np.lexsort((cols, rows))
        rows, cols = rows[o], cols[o]
    else:
        rows, cols = _sorted_unit(rng, n, 0.05)
    if variant == "adjacent_dup":
        rows = np.insert(rows, 1000, rows[1000])
        cols = np.insert(cols, 1000, cols[1000])
    elif variant == "both_directions":
        rows, cols = np.concatenate([rows, cols[:5000]]), np.concatenate([cols, rows[:5000]])
    elif variant == "loops":
        loops = np.arange(0, n, 7)
        rows, cols = np.concatenate([rows, loops]), np.concatenate([cols, loops])
    elif variant == "directed":
        directed = True
        rows, cols = np.concatenate([rows, cols[::3]]), np.concatenate([cols, rows[::3]])
    elif variant == "no_edges":
        rows, cols = rows[:0], cols[:0]
    elif variant == "tiny":
        n = 5
        rows, cols = np.array([0, 0, 1, 3], np.int64), np.array([1, 4, 2, 3], np.int64)
    elif variant == "k1":
        k = 1
    labels = rng.integers(0, k, n)
    labels[::11] = -1
    if variant == "unlabeled":
        labels[:] = -1
    _check_against_oracle(n, rows, cols, np.ones(rows.size), labels, k, directed,
                          combos=[(0, 0, 0), (1, 1, 1), (1, 0, 1), (0, 1, 0)])


# ---- configs -----------------------------------------------------------------
@pytest.mark.parametrize("idx,scale_down", [(0, 0), (1, 0), (2, 5), (3, 8), (4, 6)])
def test_configs_vs_oracle(idx, scale_down):
    from oracle import gen
    c = gen.host_config(idx, scale_down=scale_down)
    rows, cols, w, labels = c["rows"], c["cols"], c["weights"], c["labels"]
    f = c["flags"]
    combo = (int(bool(f & 1)), int(bool(f & 2)), int(bool(f & 4)))
    _check_against_oracle(c["n"], rows, cols, w, labels, c["k"], c["directed"], combos=[combo])


def test_full_cfg1_properties():
    from oracle import gen
    c = gen.host_config(1)
    edges = G.EdgeList(c["n"], c["rows"], c["cols"], c["weights"]).to_device("cuda")
    lab = G.LabelVector(c["labels"], 3)
    csr = edges.to_csr()
    assert csr.nnz == 2 * c["e"]  # SBM: no duplicates or loops, so nnz = 2E
    deg = G.degree_vector(csr, diagonal=True).cpu().numpy()
    assert same(deg, np.diff(csr.index_pointers).astype(np.float64) + 1.0)
    z = G.encode(edges, lab, G.EmbedOptions(True, True, True))
    norms = np.linalg.norm(z, axis=1)
    assert np.abs(norms - 1.0).max() <= 1e-12
    z0 = G.encode(edges, lab)
    counts = lab.class_counts()
    scaled = z0 * counts[None, :]
    assert np.abs(scaled - np.rint(scaled)).max() <= 1e-9
    assert np.rint(scaled).sum() == 2 * c["e"]


def test_encoder_plan_and_launch_count():
    from paper_2406_03726_b200 import _lib
    from oracle import gen
    c = gen.host_config(1)
    dev = torch.device("cuda")
    rows = torch.as_tensor(c["rows"], device=dev)
    cols = torch.as_tensor(c["cols"], device=dev)
    w = torch.as_tensor(c["weights"], device=dev)
    lab = torch.as_tensor(c["labels"], device=dev)
    enc = G.GeeEncoder(c["n"], c["e"], 3, False, G.EmbedOptions(True, True, True))
    lib = _lib.load()
    lib.gee_reset_launch_count()
    z1 = enc.run(rows, cols, w, lab).clone()
    assert lib.gee_launch_count() >= 5
    z2 = enc.run(rows, cols, w, lab)
    assert torch.equal(z1, z2)  # deterministic
    st, zr, _ = O.encode_edges(c["rows"], c["cols"], c["weights"], c["n"], False, c["labels"], 3, 7)
    z_close(z1.cpu().numpy(), zr)
    # the unit-weight sort path never reads a value array: same Z with weights=None
    z3 = enc.run(rows, cols, None, lab)
    z_close(z3.cpu().numpy(), zr)


@pytest.mark.parametrize("directed", [True, False])
@pytest.mark.parametrize("offset", [0, 1000, 2040, 3070])
def test_long_duplicate_runs_cross_sort_tiles(directed, offset):
    """64-bit-key radix path: a 5,000-entry run of one (row, col) pair with
    non-associative weights (its sum depends on the order) placed so it
    crosses one-sweep (3,072) and dedup (2,048) tile boundaries, mixed with
    original and reversed directions: the CSR value must be the stream-order
    sum, bit for bit."""
    rng = np.random.default_rng(offset + 7 * directed)
    n = 100_000
    m = 20_000
    rows = rng.integers(0, n, m)
    cols = rng.integers(0, n, m)
    w = 1.0 - rng.random(m)
    run = slice(3000, 8000)
    rows[run], cols[run] = 5, 9                     # row 5's entries sort first in row 5
    rows[offset:offset + 30] = 5
    cols[offset:offset + 30] = rng.integers(0, 9, 30)  # shift where the run starts in the sorted stream
    rng2 = np.random.default_rng(3)
    w[run] = rng2.choice([1e16, 1.0, -1e16, 3.0, 0.25], 5000)
    if not directed:
        rows[8000:8100], cols[8000:8100] = 9, 5     # mirrors join the (5, 9) run after the originals
        w[8000:8100] = rng2.choice([1e16, -1e16, 1.5], 100)
    for path in ("default", "sort64"):
        with assembly_path(path):
            _check_against_oracle(n, rows, cols, w, rng.integers(0, 3, n), 3, directed,
                                  combos=[(1, 1, 1), (0, 0, 0)])


class embed_flat:
    """Select the K > 8 embed variant via the library's test hook: the
    per-warp shared budget of a flat row block (0 = one warp per row)."""

    def __init__(self, nbytes, rowmax=256):
        self.nbytes, self.rowmax = nbytes, rowmax

    def __enter__(self):
        from paper_2406_03726_b200 import _lib
        lib = _lib.load()
        self.old = (lib.gee_debug_set(_lib.DEBUG_EMBED_FLAT_BYTES, self.nbytes),
                    lib.gee_debug_set(_lib.DEBUG_EMBED_FLAT_ROWMAX, self.rowmax))

    def __exit__(self, *exc):
        from paper_2406_03726_b200 import _lib
        lib = _lib.load()
        lib.gee_debug_set(_lib.DEBUG_EMBED_FLAT_BYTES, self.old[0])
        lib.gee_debug_set(_lib.DEBUG_EMBED_FLAT_ROWMAX, self.old[1])


@pytest.mark.parametrize("nbytes,rowmax", [(0, 256), (600, 1), (4096, 256), (12288, 16), (24576, 4096)])
@pytest.mark.parametrize("n,m,k,kind,directed,hub", [
    (9_000, 60_000, 9, "pos", True, (4, 0.1)),       # K just above the register path, hub > kLongRow
    (30_000, 120_000, 20, "signed", False, None),    # odd-padded tile rows (K < 32), empty rows
    (40_000, 300_000, 50, "pos", True, (5, 0.1)),    # cfg3-like K, hub row in phase 1
    (20_000, 100_000, 1000, "unit", False, (3, 0.2)),  # one row per block
])
def test_embed_flat_blocks(nbytes, rowmax, n, m, k, kind, directed, hub):
    rng = np.random.default_rng(n + k + 7)
    with embed_flat(nbytes, rowmax):
        for path in ("default", "buckets"):
            with assembly_path(path):
                _check_against_oracle(n, *_graph(rng, n, m, kind, directed, k, dup_runs=True, hub=hub), k,
                                      directed, combos=[(0, 0, 0), (1, 1, 1), (0, 1, 1), (1, 0, 0)])
