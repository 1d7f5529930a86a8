"""GpuShardOps on one B200: the per-rank kernels of the row-sharded path.

Several shards are run in one process with the collectives done by hand
(sum of histograms, concatenation of label/scale slices) -- no ranks wait
on each other -- and once through a real single-rank NCCL group."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a B200")]

from oracle import oracle as O  # noqa: E402
from test_gpu_parity import z_close  # noqa: E402

import paper_2406_03726_b200 as G  # noqa: E402
from paper_2406_03726_b200 import dist as gdist  # noqa: E402


@pytest.mark.parametrize("shards", [1, 3, 4])
@pytest.mark.parametrize("flags", [7, 1, 0])
def test_manual_shards_match_oracle(shards, flags):
    rng = np.random.default_rng(shards * 10 + flags)
    n, m, k = 3000, 40_000, 5
    rows = rng.integers(0, n, m)
    cols = rng.integers(0, n, m)
    rows[:500] = 17
    w = 1.0 - rng.random(m)
    labels = rng.integers(-1, k, n)
    dev = torch.device("cuda")
    ops = gdist.GpuShardOps(dev)
    ranges = gdist.shard_plan(rows, cols, n, False, shards)
    tr, tc, tw = (torch.as_tensor(x, device=dev) for x in (rows, cols, w))
    lab = torch.as_tensor(labels, device=dev)
    parts = []
    for rb, re in ranges:
        parts.append(ops.label_hist(lab[rb:re], k))
    counts = sum(p[1] for p in parts)                      # all-reduce
    y32 = torch.cat([p[0] for p in parts])                 # all-gather
    inv = ops.inv_counts(counts)
    csrs = []
    scale = []
    for rb, re in ranges:
        csr, sc = ops.csr_degree(*gdist.local_stream(tr, tc, tw, False, rb, re), n, flags)
        csrs.append(csr)
        scale.append(sc[rb:re])
    scale = torch.cat(scale)                               # all-gather
    z = torch.cat([ops.embed(csr, rb, re, n, y32, inv, scale, k, flags)
                   for csr, (rb, re) in zip(csrs, ranges)])
    st, zr, _ = O.encode_edges(rows, cols, w, n, False, labels, k, flags)
    pre = None
    if flags & 4:
        _, pre, _ = O.encode_edges(rows, cols, w, n, False, labels, k, flags & 3)
    z_close(z.cpu().numpy(), zr, zr_pre=pre)
    assert torch.equal(counts.cpu(), torch.as_tensor(O.class_counts(labels, k)))


def test_single_rank_nccl_group():
    import torch.distributed as dist
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(1)
        n, m, k = 2000, 20_000, 3
        rows, cols = rng.integers(0, n, m), rng.integers(0, n, m)
        labels = rng.integers(0, k, n)
        e = G.EdgeList(n, rows, cols, np.ones(m))
        z, (rb, re) = gdist.encode_sharded(e, G.LabelVector(labels, k), G.EmbedOptions(True, True, True))
        assert (rb, re) == (0, n)
        st, zr, _ = O.encode_edges(rows, cols, np.ones(m), n, False, labels, k, 7)
        z_close(z.cpu().numpy(), zr)
    finally:
        dist.destroy_process_group()


def _unit_graph(seed, n, m, k, directed, repeats):
    rng = np.random.default_rng(seed)
    rows = rng.integers(0, n, m)
    cols = rng.integers(0, n, m)
    if not directed and not repeats:
        # a simple undirected graph: i < j pairs, each once
        lo, hi = np.minimum(rows, cols), np.maximum(rows, cols)
        key = np.unique(lo[lo != hi] * n + hi[lo != hi])
        rows, cols = key // n, key % n
    if repeats:
        rows[:50] = rows[50:100]       # repeated pairs
        cols[:50] = cols[50:100]
        rows[100:120] = cols[130:150]  # pairs in both directions
        cols[100:120] = rows[130:150]
        rows[200:210] = cols[200:210]  # self loops
    labels = rng.integers(-1, k, n)
    return rows, cols, labels


@pytest.mark.parametrize("shards", [1, 2, 3, 5])
@pytest.mark.parametrize("flags", [7, 1, 0, 6])
@pytest.mark.parametrize("kind", ["simple", "repeats", "directed"])
def test_bitmap_shards_match_oracle(shards, flags, kind):
    """Unit-weight row shards on the bitmap path (gee_bitmap_shard_*), run one
    after another in this process with the degree all-gather done by hand."""
    directed = kind == "directed"
    n, m, k = 2500, 60_000, 3
    rows, cols, labels = _unit_graph(shards * 31 + flags, n, m, k, directed, kind == "repeats")
    dev = torch.device("cuda")
    ranges = gdist.shard_plan(rows, cols, n, directed, shards)
    tr, tc = (torch.as_tensor(x, device=dev) for x in (rows, cols))
    lab = torch.as_tensor(labels, device=dev)
    ops = [gdist.GpuShardOps(dev) for _ in ranges]
    streams = [gdist.local_stream(tr, tc, None, directed, rb, re) for rb, re in ranges]
    degs = [o.bm_degrees(s[0], s[1], n, rb, re, lab, k, flags) for o, s, (rb, re) in zip(ops, streams, ranges)]
    deg_all = torch.cat(degs)                                 # all-gather
    ref_len = gdist.stream_row_counts(rows, cols, n, directed)
    assert np.array_equal(deg_all.cpu().numpy(), ref_len)    # exact degrees of A
    z = torch.cat([o.bm_encode(s[0], s[1], n, rb, re, k, flags, deg_all)
                   for o, s, (rb, re) in zip(ops, streams, ranges)])
    w = np.ones(len(rows))
    st, zr, _ = O.encode_edges(rows, cols, w, n, directed, labels, k, flags)
    pre = None
    if flags & 4:
        _, pre, _ = O.encode_edges(rows, cols, w, n, directed, labels, k, flags & 3)
    z_close(z.cpu().numpy(), zr, zr_pre=pre)


def test_bitmap_shard_empty_and_out_of_range():
    dev = torch.device("cuda")
    n, k = 600, 2
    rows, cols, labels = _unit_graph(5, n, 5000, k, False, False)
    tr, tc = (torch.as_tensor(x, device=dev) for x in (rows, cols))
    lab = torch.as_tensor(labels, device=dev)
    # an empty row range
    o = gdist.GpuShardOps(dev)
    r, c, _ = gdist.local_stream(tr, tc, None, False, 300, 300)
    d = o.bm_degrees(r, c, n, 300, 300, lab, k, 7)
    assert d.numel() == 0
    z = o.bm_encode(r, c, n, 300, 300, k, 7, torch.zeros(n, dtype=torch.int32, device=dev))
    assert z.shape == (0, k)
    # entries outside the shard's rows are an edge-range error
    o = gdist.GpuShardOps(dev)
    r, c, _ = gdist.local_stream(tr, tc, None, False, 0, 300)
    o.bm_degrees(r, c, n, 0, 200, lab, k, 0)
    with pytest.raises(G.StructuralError):
        o.bm_encode(r, c, n, 0, 200, k, 0, None)


def test_single_rank_nccl_group_bitmap_path():
    import torch.distributed as dist
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rows, cols, labels = _unit_graph(9, 3000, 80_000, 3, False, False)
        e = G.EdgeList(3000, rows, cols, None)
        z, (rb, re) = gdist.encode_sharded(e, G.LabelVector(labels, 3), G.EmbedOptions(True, True, True))
        assert (rb, re) == (0, 3000)
        st, zr, _ = O.encode_edges(rows, cols, np.ones(len(rows)), 3000, False, labels, 3, 7)
        _, pre, _ = O.encode_edges(rows, cols, np.ones(len(rows)), 3000, False, labels, 3, 3)
        z_close(z.cpu().numpy(), zr, zr_pre=pre)
    finally:
        dist.destroy_process_group()


# ---- distributed CSR build: the edge shuffle kernels (k_shuffle.cu) ----------
from test_dist_gloo import partition_np, shuffle_bounds_np, shuffle_hist_np  # noqa: E402


def _shuffle_case(seed, n, m, kind, directed):
    rng = np.random.default_rng(seed)
    rows = rng.integers(0, n, m)
    cols = rng.integers(0, n, m)
    rows[: m // 10] = 3  # a hub row (R-MAT-like skew) and self loops
    cols[: m // 50] = 3
    if kind == "f64":
        w = 1.0 - rng.random(m)
    elif kind == "f32":
        w = (1.0 - rng.random(m, dtype=np.float32)).astype(np.float32)
    else:
        w = None
    return rows, cols, w


@pytest.mark.parametrize("n,m,kind,directed,world", [
    (5000, 60_000, "f64", False, 3), (5000, 60_000, "f32", True, 5), (40_000, 200_000, "unit", False, 8),
    (100, 0, "f64", False, 2), (20_000, 100_000, "f64", True, 1), (70_000, 50_000, "f32", False, 16)])
def test_shuffle_kernels_match_restatement(n, m, kind, directed, world):
    """gee_shuffle_row_hist / gee_shuffle_bounds / gee_partition are bit-exact
    against the numpy restatements the gloo tests drive the orchestration with,
    and the per-destination exchange order reproduces local_stream()."""
    rows, cols, w = _shuffle_case(n + m + world, n, m, kind, directed)
    ops = gdist.GpuShardOps("cuda")
    cuts = np.linspace(0, m, world + 1).astype(np.int64)
    if world > 1:
        cuts[1] = cuts[0]  # an empty slice
    dev = torch.device("cuda")
    hist = None
    for a, b in zip(cuts, cuts[1:]):
        r = torch.as_tensor(rows[a:b], device=dev)
        c = torch.as_tensor(cols[a:b], device=dev)
        h = ops.row_hist(r, c, n, directed).cpu().numpy()
        assert np.array_equal(h, shuffle_hist_np(rows[a:b], cols[a:b], n, directed))
        hist = h if hist is None else hist + h
    bounds = ops.shuffle_bounds(torch.as_tensor(hist, device=dev), n, world)
    assert np.array_equal(bounds.cpu().numpy(), shuffle_bounds_np(hist, n, world))
    sent = []
    for a, b in zip(cuts, cuts[1:]):
        r = torch.as_tensor(rows[a:b], device=dev)
        c = torch.as_tensor(cols[a:b], device=dev)
        ww = None if w is None else torch.as_tensor(w[a:b], device=dev)
        gr, gc, gw, cnt = ops.partition(r, c, ww, directed, bounds, world)
        er, ec, ew, ecnt = partition_np(rows[a:b], cols[a:b], None if w is None else w[a:b], directed,
                                        bounds.cpu().numpy(), world)
        tot = int(sum(cnt))
        assert cnt == ecnt.tolist()
        assert np.array_equal(gr[:tot].cpu().numpy(), er) and np.array_equal(gc[:tot].cpu().numpy(), ec)
        if w is not None:
            assert gw.dtype == ww.dtype and np.array_equal(gw[:tot].cpu().numpy(), ew)
        sent.append((gr[:tot].cpu().numpy(), gc[:tot].cpu().numpy(),
                     None if w is None else gw[:tot].cpu().numpy(), np.asarray(cnt)))
    bnd = bounds.cpu().numpy()
    for d in range(world):
        seq = []
        for half in (0, 1):
            for r, c, ww, cnt in sent:
                off = np.concatenate([[0], np.cumsum(cnt)])
                lo, hi = off[half * world + d], off[half * world + d + 1]
                seq.append((r[lo:hi], c[lo:hi], None if ww is None else ww[lo:hi]))
        er, ec, ew = gdist.local_stream(rows, cols, w, directed, int(bnd[d]), int(bnd[d + 1]))
        assert np.array_equal(np.concatenate([x[0] for x in seq]), er)
        assert np.array_equal(np.concatenate([x[1] for x in seq]), ec)
        if w is not None:
            assert np.array_equal(np.concatenate([x[2] for x in seq]), ew)


@pytest.mark.parametrize("kind,k,flags", [("f32", 50, 7), ("unit", 3, 7), ("f64", 20, 1)])
def test_single_rank_nccl_group_edge_shuffle(kind, k, flags):
    """encode_distributed through a real NCCL group (all-reduce of the row
    histogram, all-to-all of the partitioned slice) against the oracle."""
    import torch.distributed as dist
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        n, m = 3000, 30_000
        rows, cols, w = _shuffle_case(k + flags, n, m, kind, False)
        labels = np.random.default_rng(k).integers(-1, k, n)
        w_in = np.ones(m) if w is None else w
        z, (rb, re) = gdist.encode_distributed(rows, cols, w_in, n, False, labels, k,
                                               G.EmbedOptions(bool(flags & 1), bool(flags & 2), bool(flags & 4)))
        assert (rb, re) == (0, n)
        st, zr, _ = O.encode_edges(rows, cols, np.asarray(w_in, np.float64), n, False, labels, k, flags)
        assert st == O.OK
        z_close(z.cpu().numpy(), zr)
    finally:
        dist.destroy_process_group()


# ---- the stream path per row shard (gee_stream_shard_*) ---------------------
@pytest.mark.parametrize("shards", [1, 2, 5])
@pytest.mark.parametrize("flags,directed,kind", [(7, False, "f64"), (5, True, "f32"), (3, False, "unit"),
                                                 (0, True, "f64")])
def test_stream_shards_match_oracle(shards, flags, directed, kind):
    """Every shard runs phase 1 (its rows' degrees), the degree vectors are
    concatenated by hand (the all-gather), then phase 2 per shard."""
    rng = np.random.default_rng(shards * 100 + flags)
    n, m, k = 5000, 60_000, 20
    rows = rng.integers(0, n, m)
    cols = rng.integers(0, n, m)
    rows[:3000] = 11  # a hub: split buckets in its shard
    w = np.ones(m) if kind == "unit" else (1.0 - rng.random(m))
    if kind == "f32":
        w = w.astype(np.float32)
    labels = rng.integers(-1, k, n)
    dev = torch.device("cuda")
    ranges = gdist.shard_plan(rows, cols, n, directed, shards)
    tr, tc = torch.as_tensor(rows, device=dev), torch.as_tensor(cols, device=dev)
    tw = None if kind == "unit" else torch.as_tensor(w, device=dev)
    lab = torch.as_tensor(labels, device=dev)
    opss, streams, degs = [], [], []
    for rb, re in ranges:
        ops = gdist.GpuShardOps(dev)
        st = gdist.local_stream(tr, tc, tw, directed, rb, re)
        ops.st_prepare(*st, n, rb, re, k, flags)
        degs.append(ops.st_degrees(*st, lab).clone())
        opss.append(ops)
        streams.append(st)
    deg_all = torch.cat(degs)                              # all-gather
    z = torch.cat([ops.st_encode(deg_all if flags & 1 else None) for ops in opss])
    for ops in opss:
        ops.st_check()
    st_, zr, _ = O.encode_edges(rows, cols, np.asarray(w, np.float64), n, directed, labels, k, flags)
    assert st_ == O.OK
    z_close(z.cpu().numpy(), zr)


def test_single_rank_nccl_group_stream_path():
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        rng = np.random.default_rng(3)
        n, m, k = 20000, 100_000, 50
        rows = rng.integers(0, n, m)
        cols = rng.integers(0, n, m)
        w = (1.0 - rng.random(m)).astype(np.float32)
        labels = rng.integers(0, k, n)
        e = G.EdgeList(n, rows, cols, w, directed=True)
        lab = G.LabelVector(labels, k)
        opts = G.EmbedOptions(True, True, True)
        z, (rb, re) = gdist.encode_sharded(e, lab, opts)
        assert (rb, re) == (0, n)
        st, zr, _ = O.encode_edges(rows, cols, w.astype(np.float64), n, True, labels, k, 7)
        z_close(z.cpu().numpy(), zr)
    finally:
        dist.destroy_process_group()
