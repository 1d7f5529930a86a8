"""Multi-GPU row sharding, exercised on CPU with the gloo backend (world 2).

dist.encode_rows runs the real orchestration (all-reduce of the class
histogram, all-gather of labels and of the Laplacian scale, row-range
embed); the per-rank compute is an oracle-backed stand-in defined here (the
product uses GpuShardOps).  Shard-count invariance: the assembled Z must be
BITWISE equal to the unsharded reference pipeline, because every row is
computed from exactly the same entries, degrees and scales.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2406_03726_b200 import dist as gdist

LAP, DIAG, CORR = 1, 2, 4


def shuffle_hist_np(rows, cols, n, directed, max_buckets=16384):
    """Stream entries per coarse row bucket floor(r * B / n), B = min(n, 16384)."""
    nb = min(n, max_buckets)
    b = (rows.astype(np.int64) * nb) // n
    h = np.bincount(b, minlength=nb)
    if not directed:
        off = rows != cols
        h = h + np.bincount((cols[off].astype(np.int64) * nb) // n, minlength=nb)
    return h.astype(np.int64)


def shuffle_bounds_np(hist, n, world):
    """dist.row_ranges on bucket granularity (bucket b starts at row ceil(b n / B))."""
    nb = len(hist)
    total = int(hist.sum())
    bounds = [0]
    run, b = 0, 0
    for p in range(1, world):
        target = total * p // world
        while b < nb and run < target:
            run += int(hist[b])
            b += 1
        row = min(max(-(-b * n // nb), bounds[-1]), n)
        bounds.append(row)
    bounds.append(n)
    return np.array(bounds, np.int64)


def partition_np(rows, cols, w, directed, bounds, world):
    """Stable [half][dest] partition: originals by row, mirrored off-diagonals
    (as (col, row)) by column, each bucket in slice order."""
    dest_o = np.searchsorted(bounds[1:-1], rows, side="right")
    parts_r, parts_c, parts_w, counts = [], [], [], []
    for half in (0, 1):
        if half == 0:
            rr, cc, ww, dd = rows, cols, w, dest_o
        else:
            m = (rows != cols) if not directed else np.zeros(rows.size, bool)
            rr, cc = cols[m], rows[m]
            ww = None if w is None else w[m]
            dd = np.searchsorted(bounds[1:-1], rr, side="right")
        for d in range(world):
            sel = dd == d
            parts_r.append(rr[sel])
            parts_c.append(cc[sel])
            if w is not None:
                parts_w.append(ww[sel])
            counts.append(int(sel.sum()))
    cat = lambda xs, dt: np.concatenate(xs) if xs else np.zeros(0, dt)
    return (cat(parts_r, np.int64), cat(parts_c, np.int64),
            None if w is None else cat(parts_w, w.dtype), np.array(counts, np.int64))


class OracleShardOps:
    """CPU stand-in for GpuShardOps built from the oracle (test only)."""

    dev = torch.device("cpu")

    def label_hist(self, labels_slice, k):
        lab = labels_slice.numpy()
        return torch.as_tensor(lab.astype(np.int32)), torch.as_tensor(O.class_counts(lab, k))

    def inv_counts(self, counts):
        c = counts.to(torch.float64)
        return torch.where(c > 0, 1.0 / c, torch.zeros_like(c))

    def csr_degree(self, r, c, w, n, flags):
        w64 = np.ones(r.numel()) if w is None else w.numpy().astype(np.float64)
        ip, cc, cv = O.coo_to_csr(r.numpy(), c.numpy(), w64, n, n)
        if flags & DIAG:
            dip, _, dcv = O.add_identity(ip, cc, cv, n)
            deg = O.degree(dip, dcv, n)
        else:
            deg = O.degree(ip, cv, n)
        scale = np.where(deg > 0, 1.0 / np.sqrt(np.where(deg > 0, deg, 1.0)), 0.0)
        return (ip, cc, cv), torch.as_tensor(scale)

    def embed(self, csr, rb, re, n, y32, inv, scale, k, flags):
        ip, cc, cv = csr
        if flags & DIAG:
            ip, cc, cv = O.add_identity(ip, cc, cv, n)
        if flags & LAP:
            s = scale.numpy()
            rid = np.repeat(np.arange(n), np.diff(ip))
            v = cv * s[rid] * s[cc]
            keep = v != 0.0
            ptr = np.zeros(n + 1, np.int64)
            np.cumsum(np.bincount(rid[keep], minlength=n), out=ptr[1:])
            ip, cc, cv = ptr, cc[keep], v[keep]
        z = O.spmm_onehot_dense(ip, cc, cv, y32.numpy().astype(np.int64), k)[rb:re]
        if flags & CORR:
            z = O.correlate_rows(z)
        return torch.as_tensor(z)

    # bitmap path: phase 1 = stream lengths of the local rows, phase 2 = Z
    # rows from the local stream and the gathered degree vector
    def bm_degrees(self, r, c, n, rb, re, labels, k, flags):
        self._labels = labels.numpy().astype(np.int64)
        return torch.as_tensor(np.bincount(r.numpy() - rb, minlength=re - rb).astype(np.int32))

    # stream path: phase 1 = raw degrees of the local rows, phase 2 = Z rows
    # from the gathered degree vector (the oracle's CSR of the local stream)
    def st_prepare(self, r, c, w, n, rb, re, k, flags):
        self._st = dict(e=int(r.numel()), rb=rb, re=re, n=n, k=k, flags=flags, stream=(r, c, w))
        return self._st

    def st_degrees(self, r, c, w, labels):
        p = self._st
        self._labels = labels.numpy().astype(np.int64)
        w64 = np.ones(r.numel()) if w is None else w.numpy().astype(np.float64)
        ip, cc, cv = O.coo_to_csr(r.numpy(), c.numpy(), w64, p["n"], p["n"])
        p["csr"] = (ip, cc, cv)
        return torch.as_tensor(O.degree(ip, cv, p["n"])[p["rb"]:p["re"]])

    def st_encode(self, deg_all, z=None):
        p = self._st
        n, k, flags = p["n"], p["k"], p["flags"]
        scale = None
        if flags & LAP:
            if flags & DIAG:
                ip, cc, cv = p["csr"]
                aug = O.add_identity(ip, cc, cv, n)
                local = O.degree(aug[0], aug[2], n)[p["rb"]:p["re"]]
                deg = deg_all.numpy().astype(np.float64).copy()
                # the gathered degrees are raw; A+I adds the diagonal term as the
                # reference merges it (v_rr + 1.0 at its sorted position)
                deg = np.where(np.arange(n) >= 0, deg + 1.0, deg)
                deg[p["rb"]:p["re"]] = local
            else:
                deg = deg_all.numpy().astype(np.float64)
            scale = torch.as_tensor(np.where(deg > 0, 1.0 / np.sqrt(np.where(deg > 0, deg, 1.0)), 0.0))
        y32 = torch.as_tensor(self._labels.astype(np.int32))
        inv = self.inv_counts(torch.as_tensor(O.class_counts(self._labels, k)))
        return self.embed(p["csr"], p["rb"], p["re"], n, y32, inv, scale, k, flags)

    def st_check(self):
        pass

    @staticmethod
    def bitmap_ok(n, k, weighted):
        return not weighted and 1 <= n <= 16384 and 1 <= k <= 8

    # edge shuffle: numpy restatements of k_shuffle.cu (tests/test_gpu_dist.py
    # pins the kernels against these)
    def row_hist(self, rows, cols, n, directed):
        return torch.as_tensor(shuffle_hist_np(rows.numpy(), cols.numpy(), n, directed))

    def shuffle_bounds(self, hist, n, world):
        return torch.as_tensor(shuffle_bounds_np(hist.numpy(), n, world))

    def partition(self, rows, cols, w, directed, bounds, world):
        r, c, ww, counts = partition_np(rows.numpy(), cols.numpy(), None if w is None else w.numpy(), directed,
                                        bounds.numpy(), world)
        return (torch.as_tensor(r), torch.as_tensor(c), None if ww is None else torch.as_tensor(ww),
                counts.tolist())

    def bm_encode(self, r, c, n, rb, re, k, flags, deg_all, check=True):
        rr = r.numpy()
        assert ((rr >= rb) & (rr < re)).all()
        ip, cc, cv = O.coo_to_csr(rr, c.numpy(), np.ones(rr.size), n, n)
        scale = None
        if flags & LAP:
            deg = deg_all.numpy().astype(np.float64) + (1.0 if flags & DIAG else 0.0)
            scale = torch.as_tensor(np.where(deg > 0, 1.0 / np.sqrt(np.where(deg > 0, deg, 1.0)), 0.0))
        y32 = torch.as_tensor(self._labels.astype(np.int32))
        inv = self.inv_counts(torch.as_tensor(O.class_counts(self._labels, k)))
        return self.embed((ip, cc, cv), rb, re, n, y32, inv, scale, k, flags)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _graph(seed, n=300, m=2000, k=4, directed=False, weighted=True):
    rng = np.random.default_rng(seed)
    rows = rng.integers(0, n, m)
    cols = rng.integers(0, n, m)
    rows[:40] = 7  # a hub row and duplicate coordinates
    cols[:10] = 11
    w = (1.0 - rng.random(m)) if weighted else np.ones(m)
    labels = rng.integers(-1, k, n)
    return n, rows, cols, w, labels, k, directed


def _worker(rank, world, port, case, flags, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, rows, cols, w, labels, k, directed = case
        ranges = gdist.shard_plan(rows, cols, n, directed, world)
        rb, re = ranges[rank]
        r, c, ww = gdist.local_stream(torch.as_tensor(rows), torch.as_tensor(cols), torch.as_tensor(w),
                                      directed, rb, re)
        z = gdist.encode_rows(OracleShardOps(), (r, c, ww), torch.as_tensor(labels), n, k, flags, ranges,
                              rank)
        full = gdist.gather_z(z, ranges)
        if rank == 0:
            out.put(full.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("flags", [0, LAP | DIAG | CORR, LAP, DIAG | CORR])
@pytest.mark.parametrize("directed", [False, True])
def test_two_rank_sharding_is_bitwise_shard_invariant(flags, directed):
    case = _graph(3 + flags + directed, directed=directed)
    n, rows, cols, w, labels, k, _ = case
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_worker, args=(2, _free_port(), case, flags, q), nprocs=2, join=True)
    z = q.get(timeout=60)
    st, zr, _ = O.encode_edges(rows, cols, w, n, directed, labels, k, flags)
    assert st == O.OK
    assert z.shape == zr.shape and np.array_equal(z, zr)


def _bm_worker(rank, world, port, case, flags, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, rows, cols, _, labels, k, directed = case
        ranges = gdist.shard_plan(rows, cols, n, directed, world)
        stream = gdist.local_stream(torch.as_tensor(rows), torch.as_tensor(cols), None, directed, *ranges[rank])
        z = gdist.encode_rows_bitmap(OracleShardOps(), stream, torch.as_tensor(labels), n, k, flags, ranges,
                                     rank)
        full = gdist.gather_z(z, ranges)
        if rank == 0:
            out.put(full.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("flags", [0, LAP | DIAG | CORR, LAP])
@pytest.mark.parametrize("directed", [False, True])
def test_two_rank_bitmap_path_degree_allgather(flags, directed):
    """Unit-weight path: only the degree vector is exchanged; Z assembled
    from the two shards equals the unsharded oracle bitwise."""
    case = _graph(11 + flags + directed, directed=directed, weighted=False, k=3)
    n, rows, cols, w, labels, k, _ = case
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_bm_worker, args=(2, _free_port(), case, flags, q), nprocs=2, join=True)
    z = q.get(timeout=60)
    st, zr, _ = O.encode_edges(rows, cols, w, n, directed, labels, k, flags)
    assert st == O.OK
    assert z.shape == zr.shape and np.array_equal(z, zr)


def test_row_ranges_balance_stream_entries():
    counts = np.array([5, 0, 0, 100, 1, 1, 1, 1, 50, 2])
    rr = gdist.row_ranges(counts, 3)
    assert rr[0][0] == 0 and rr[-1][1] == len(counts)
    assert all(a[1] == b[0] for a, b in zip(rr, rr[1:]))
    rr1 = gdist.row_ranges(counts, 1)
    assert rr1 == [(0, len(counts))]


def test_local_stream_keeps_stream_order():
    rows = np.array([0, 2, 1, 2, 0])
    cols = np.array([2, 1, 1, 0, 2])
    w = np.array([1.0, 2.0, 3.0, 4.0, 5.0])
    r, c, ww = gdist.local_stream(rows, cols, w, False, 2, 3)
    # originals with row 2 (e=1, e=3) first, then reversed off-diagonals with col 2 (e=0, e=4)
    assert r.tolist() == [2, 2, 2, 2] and c.tolist() == [1, 0, 0, 0]
    assert ww.tolist() == [2.0, 4.0, 1.0, 5.0]
    counts = gdist.stream_row_counts(rows, cols, 3, False)
    # 5 originals + 4 reversed off-diagonals (e=2 is a self loop, counted once)
    assert counts.tolist() == [3, 2, 4] and counts.sum() == 9


def _slice_worker(rank, world, port, case, flags, cuts, out):
    """Every rank holds ONLY its contiguous slice of the original edge list."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, rows, cols, w, labels, k, directed = case
        lo, hi = cuts[rank], cuts[rank + 1]
        z, (rb, re) = gdist.encode_distributed(torch.as_tensor(rows[lo:hi]), torch.as_tensor(cols[lo:hi]),
                                               torch.as_tensor(w[lo:hi]), n, directed, torch.as_tensor(labels),
                                               k, _opts(flags), ops=OracleShardOps())
        ranges = [None] * world
        dist.all_gather_object(ranges, (rb, re))
        full = gdist.gather_z(z, ranges)
        if rank == 0:
            out.put(full.numpy())
    finally:
        dist.destroy_process_group()


def _opts(flags):
    from paper_2406_03726_b200.graph import EmbedOptions
    return EmbedOptions(laplacian=bool(flags & LAP), diagonal=bool(flags & DIAG), correlation=bool(flags & CORR))


@pytest.mark.parametrize("weighted,directed,world,flags", [
    (True, False, 3, LAP | DIAG | CORR), (False, False, 2, LAP | DIAG | CORR),
    (True, True, 2, LAP), (False, True, 3, LAP | CORR)])
def test_edge_shuffle_from_partitioned_slices(weighted, directed, world, flags):
    """Distributed CSR build: ranks start from uneven slices of the edge list
    (one of them empty in the 3-rank cases); the all-to-all edge shuffle must
    reproduce the unsharded Z bitwise (weighted: CSR path; unit weights with
    n <= 16384 and k <= 3: the bitmap path)."""
    case = _graph(21 + flags + 2 * directed + 4 * weighted, directed=directed, weighted=weighted, k=3)
    n, rows, cols, w, labels, k, _ = case
    m = rows.size
    cuts = [0, m // 3, m] if world == 2 else [0, 700, 700, m]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_slice_worker, args=(world, _free_port(), case, flags, cuts, q), nprocs=world, join=True)
    z = q.get(timeout=60)
    st, zr, _ = O.encode_edges(rows, cols, w, n, directed, labels, k, flags)
    assert st == O.OK
    assert z.shape == zr.shape and np.array_equal(z, zr)


def test_partition_np_matches_local_stream():
    """The restated partition + exchange order equals local_stream() on every
    destination (the property the shuffle's bitwise invariance rests on)."""
    n, rows, cols, w, labels, k, directed = _graph(5, directed=False)
    cuts = [0, 500, 1200, rows.size]
    world = 3
    hist = sum(shuffle_hist_np(rows[a:b], cols[a:b], n, directed) for a, b in zip(cuts, cuts[1:]))
    bounds = shuffle_bounds_np(hist, n, world)
    full_counts = gdist.stream_row_counts(rows, cols, n, directed)
    assert hist.sum() == full_counts.sum()
    sent = [partition_np(rows[a:b], cols[a:b], w[a:b], directed, bounds, world) for a, b in zip(cuts, cuts[1:])]
    for d in range(world):
        got = {0: [], 1: []}
        for r, c, ww, cnt in sent:
            off = np.concatenate([[0], np.cumsum(cnt)])
            for half in (0, 1):
                b = half * world + d
                got[half].append((r[off[b]:off[b + 1]], c[off[b]:off[b + 1]], ww[off[b]:off[b + 1]]))
        seq = got[0] + got[1]
        r = np.concatenate([x[0] for x in seq])
        c = np.concatenate([x[1] for x in seq])
        ww = np.concatenate([x[2] for x in seq])
        er, ec, ew = gdist.local_stream(rows, cols, w, directed, int(bounds[d]), int(bounds[d + 1]))
        assert np.array_equal(r, er) and np.array_equal(c, ec) and np.array_equal(ww, ew)


def _st_worker(rank, world, port, case, flags, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, rows, cols, w, labels, k, directed = case
        ranges = gdist.shard_plan(rows, cols, n, directed, world)
        stream = gdist.local_stream(torch.as_tensor(rows), torch.as_tensor(cols), torch.as_tensor(w), directed,
                                    *ranges[rank])
        z = gdist.encode_rows_stream(OracleShardOps(), stream, torch.as_tensor(labels), n, k, flags, ranges, rank)
        full = gdist.gather_z(z, ranges)
        if rank == 0:
            out.put(full.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("flags", [LAP | DIAG | CORR, LAP | CORR, 0])
def test_stream_path_degree_allgather(world, flags):
    """Stream path orchestration: phase 1 per rank, ALL-GATHER of the f64
    degree vector, phase 2 per rank; Z assembled from the shards matches the
    unsharded oracle within the north_star's 1e-12 (the gathered degrees are
    raw sums; A+I's 1.0 is added after the exchange, which the reference
    merges into the diagonal entry instead -- a rounding-level difference)."""
    case = _graph(21 + flags + world, directed=True)
    n, rows, cols, w, labels, k, directed = case
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_st_worker, args=(world, _free_port(), case, flags, q), nprocs=world, join=True)
    z = q.get(timeout=60)
    st, zr, _ = O.encode_edges(rows, cols, w, n, directed, labels, k, flags)
    assert st == O.OK
    rown = np.sqrt((zr * zr).sum(axis=1, keepdims=True))
    assert z.shape == zr.shape and (np.abs(z - zr) <= 1e-12 * np.maximum(np.abs(zr), rown) + 1e-15).all()
