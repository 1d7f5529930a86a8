"""Row-sharded multi-GPU encode: one process per GPU, torch.distributed.

Rows of Z are independent once every rank knows the per-node tables, so the
graph is split into P contiguous row ranges holding equal numbers of stream
entries.  Rank p owns rows [rb, re):

  1. its slice of the symmetrised stream -- the entries whose row falls in
     [rb, re), kept in stream order ([originals..., reversed...],
     graph_io.py:82-88), so duplicate sums and hence the CSR are bitwise
     identical to the unsharded build (shard-count invariance);
  2. K1 on its label slice, then ALL-REDUCE(sum) of the class histogram
     (int64, K) and ALL-GATHER of the int32 labels (every column's class is
     needed by the embed);
  3. K2+K3 on its stream slice: CSR rows and their degrees (a row's degree
     depends only on its own entries);
  4. under Laplacian, ALL-GATHER of the scale vector s = d^-1/2 (f64, N) --
     the one real exchange of the algorithm: row r needs s_j of every
     neighbour j, owned by other ranks;
  5. K4 over rows [rb, re); Z stays row-sharded (gather_z collects it).

Unit-weight graphs of at most 16384 nodes and K <= 8 (configs 0/1) take the
bitmap path instead (encode_rows_bitmap): each rank sets the adjacency bits of
its own rows only (no transpose pass: its slice already holds both
directions), reports its rows' degrees, and after ONE all-gather of those
degrees (uint32, N; only under the Laplacian) runs the node table and the
tensor-core product over its row tiles.  Labels are replicated, so the class
histogram needs no all-reduce there.

The collectives are torch.distributed calls (NCCL over NVLink on the GPU
box; gloo in the CPU tests).  The per-rank compute is an object with four
methods; the product uses GpuShardOps (libgee).  tests/test_dist_gloo.py
drives the same orchestration with an oracle-backed stand-in to prove
shard-count invariance on CPU -- the product never constructs one.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _device, _lib


# ---------------------------------------------------------------------------
# host-side partitioning (data distribution, outside the timed region)
# ---------------------------------------------------------------------------
def stream_row_counts(rows, cols, n: int, directed: bool) -> np.ndarray:
    """Entries per row of the symmetrised stream (numpy, int64[n])."""
    rows = _np(rows)
    cols = _np(cols)
    cnt = np.bincount(rows, minlength=n)
    if not directed:
        off = rows != cols
        cnt = cnt + np.bincount(cols[off], minlength=n)
    return cnt.astype(np.int64)


def row_ranges(row_counts, world: int) -> list[tuple[int, int]]:
    """`world` contiguous row ranges with (nearly) equal stream entries."""
    c = np.concatenate([[0], np.cumsum(np.asarray(row_counts, dtype=np.int64))])
    n = len(c) - 1
    total = int(c[-1])
    bounds = [0]
    for p in range(1, world):
        target = total * p // world
        b = int(np.searchsorted(c, target, side="left"))
        bounds.append(min(max(b, bounds[-1]), n))
    bounds.append(n)
    return [(bounds[p], bounds[p + 1]) for p in range(world)]


def local_stream(rows, cols, weights, directed: bool, rb: int, re: int):
    """Stream entries whose row is in [rb, re), in stream order, as a
    directed edge list (global node ids)."""
    is_t = isinstance(rows, torch.Tensor)
    cat = torch.cat if is_t else np.concatenate
    in1 = (rows >= rb) & (rows < re)
    r_parts, c_parts, w_parts = [rows[in1]], [cols[in1]], []
    if weights is not None:
        w_parts.append(weights[in1])
    if not directed:
        in2 = (cols >= rb) & (cols < re) & (rows != cols)
        r_parts.append(cols[in2])
        c_parts.append(rows[in2])
        if weights is not None:
            w_parts.append(weights[in2])
    r = cat(r_parts)
    c = cat(c_parts)
    w = cat(w_parts) if weights is not None else None
    return r, c, w


def _np(x):
    return x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


# ---------------------------------------------------------------------------
# collectives (equal-size padded all-gather works for gloo and NCCL alike)
# ---------------------------------------------------------------------------
def all_gather_ranges(local: torch.Tensor, ranges, group=None) -> torch.Tensor:
    """Concatenate every rank's slice (lengths re-rb) into one full vector."""
    world = len(ranges)
    width = max(re - rb for rb, re in ranges)
    buf = torch.zeros(width, dtype=local.dtype, device=local.device)
    buf[: local.numel()] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([parts[p][: re - rb] for p, (rb, re) in enumerate(ranges)])


# ---------------------------------------------------------------------------
# per-rank compute on the GPU (libgee)
# ---------------------------------------------------------------------------
class GpuShardOps:
    """K1..K4 for one row shard through the C ABI."""

    def __init__(self, device):
        self.dev = torch.device(device)
        self.lib = _lib.load()

    def label_hist(self, labels_slice, k):
        lab = _device.to_device(labels_slice, torch.int64, self.dev)
        n = lab.numel()
        y32 = torch.empty(max(n, 1), dtype=torch.int32, device=self.dev)
        counts = torch.empty(k, dtype=torch.int64, device=self.dev)
        inv = torch.empty(k, dtype=torch.float64, device=self.dev)
        err = _device.error_word(self.dev)
        _lib.check(self.lib.gee_label_hist(_device.ptr(lab), n, k, _device.ptr(y32), _device.ptr(counts),
                                           _device.ptr(inv), _device.ptr(err), _device.stream_handle()))
        self._err = err
        return y32[:n], counts

    def inv_counts(self, counts):
        inv = torch.empty(counts.numel(), dtype=torch.float64, device=self.dev)
        _lib.check(self.lib.gee_inv_counts(_device.ptr(counts), counts.numel(), _device.ptr(inv),
                                           _device.stream_handle()))
        return inv

    def csr_degree(self, r, c, w, n, flags):
        """CSR of the shard's rows (global ids, other rows empty) + degrees/scale."""
        e = int(r.numel())
        if w is None:
            wt = _lib.W_UNIT
        else:
            wt = _lib.W_F32 if w.dtype == torch.float32 else _lib.W_F64
        cap = max(e, 1)
        row_ptr = torch.empty(n + 1, dtype=torch.int64, device=self.dev)
        col = torch.empty(cap, dtype=torch.int32, device=self.dev)
        val = torch.empty(cap, dtype=torch.float64, device=self.dev)
        deg = torch.empty(n, dtype=torch.float64, device=self.dev)
        scale = torch.empty(n, dtype=torch.float64, device=self.dev)
        err = _device.error_word(self.dev)
        dflags = (_lib.LAPLACIAN | (flags & _lib.DIAGONAL)) if flags & _lib.LAPLACIAN else 0
        nb = _lib.size_query(self.lib.gee_csr_build_workspace, e, n, n, 1)
        ws = _device.WORKSPACE.get(nb, self.dev)
        _lib.check(self.lib.gee_csr_build(
            _device.ptr(r), _device.ptr(c), _device.ptr(w), wt, e, n, n, 1, 1, _device.ptr(row_ptr), None,
            _device.ptr(col), _device.ptr(val), None, dflags, _device.ptr(deg), _device.ptr(scale),
            _device.ptr(ws), ws.numel(), _device.ptr(err), _device.stream_handle()))
        self._err2 = err
        return (row_ptr, col, val), scale

    def embed(self, csr, rb, re, n, y32, inv, scale, k, flags):
        row_ptr, col, val = csr
        z = torch.empty((re - rb, k), dtype=torch.float64, device=self.dev)
        err = _device.error_word(self.dev)
        nb = _lib.size_query(self.lib.gee_embed_workspace, re - rb, n)
        ws = torch.empty(max(nb, 256), dtype=torch.uint8, device=self.dev)
        _lib.check(self.lib.gee_embed(
            _device.ptr(row_ptr), None, _device.ptr(col), _device.ptr(val), rb, re, n, _device.ptr(y32),
            _device.ptr(inv), _device.ptr(scale) if flags & _lib.LAPLACIAN else None, k, flags, _device.ptr(z), k,
            _device.ptr(ws), ws.numel(), _device.ptr(err), _device.stream_handle()))
        bits = int(self._err.item()) | int(self._err2.item()) | int(err.item())
        _lib.raise_device_errors(bits, "sharded encode")
        return z

    # -- stream path (unit or non-negative weights; k_stream.cu) -------------
    def st_prepare(self, r, c, w, n, rb, re, k, flags):
        """Plan the row shard's stream encode (workspace sized once)."""
        e = int(r.numel())
        wt = _lib.W_UNIT if w is None else (_lib.W_F32 if w.dtype == torch.float32 else _lib.W_F64)
        f = flags | _lib.NONNEG
        nb = _lib.size_query(self.lib.gee_stream_shard_workspace, e, n, rb, re, k, wt, f)
        self._st = dict(e=e, wt=wt, n=n, rb=rb, re=re, k=k, flags=f,
                        ws=torch.empty(max(nb, 256), dtype=torch.uint8, device=self.dev),
                        deg=torch.empty(max(re - rb, 1), dtype=torch.float64, device=self.dev),
                        err=_device.error_word(self.dev))
        return self._st

    def st_degrees(self, r, c, w, labels):
        """Phase 1: partition the shard's entries, degrees of its rows (raw, f64)."""
        p = self._st
        _lib.check(self.lib.gee_stream_shard_degrees(
            _device.ptr(r), _device.ptr(c), _device.ptr(w), p["wt"], p["e"], p["n"], p["rb"], p["re"],
            _device.ptr(labels), p["k"], p["flags"], _device.ptr(p["deg"]), _device.ptr(p["ws"]), p["ws"].numel(),
            _device.ptr(p["err"]), _device.stream_handle()))
        return p["deg"][: p["re"] - p["rb"]]

    def st_encode(self, deg_all, z=None):
        """Phase 2: node table from the gathered degrees, Z of the shard's rows."""
        p = self._st
        if z is None:
            z = torch.empty((p["re"] - p["rb"], p["k"]), dtype=torch.float64, device=self.dev)
        _lib.check(self.lib.gee_stream_shard_encode(
            p["wt"], p["e"], p["n"], p["rb"], p["re"], p["k"], p["flags"], _device.ptr(deg_all), _device.ptr(z),
            _device.ptr(p["ws"]), p["ws"].numel(), _device.ptr(p["err"]), _device.stream_handle()))
        return z

    def st_check(self):
        _lib.raise_device_errors(int(self._st["err"].item()), "sharded stream encode")

    # -- bitmap path (unit weights, n <= 16384, k <= 8) ----------------------
    BITMAP_MAX_NODES = 16384

    @classmethod
    def bitmap_ok(cls, n, k, weighted):
        return not weighted and 1 <= n <= cls.BITMAP_MAX_NODES and 1 <= k <= 8

    def bm_degrees(self, r, c, n, rb, re, labels, k, flags):
        """Phase 1: local bitmap rows -> int32[re-rb] stream lengths (the
        rows' unit-weight degrees).  labels: all n (replicated)."""
        e = int(r.numel())
        nb = _lib.size_query(self.lib.gee_bitmap_shard_workspace, e, n, rb, re, k)
        ws = getattr(self, "_bm_ws", None)
        if ws is None or ws.numel() < nb:
            ws = self._bm_ws = torch.empty(max(nb, 256), dtype=torch.uint8, device=self.dev)
        self._bm_err = _device.error_word(self.dev)
        deg = torch.empty(max(re - rb, 1), dtype=torch.int32, device=self.dev)
        _lib.check(self.lib.gee_bitmap_shard_degrees(
            _device.ptr(r), _device.ptr(c), e, n, rb, re, _device.ptr(labels), k, flags, _device.ptr(deg),
            _device.ptr(ws), ws.numel(), _device.ptr(self._bm_err), _device.stream_handle()))
        return deg[: re - rb]

    def bm_encode(self, r, c, n, rb, re, k, flags, deg_all, check=True):
        """Phase 2 (after bm_degrees on this object): Z[rb:re]."""
        e = int(r.numel())
        z = torch.empty((re - rb, k), dtype=torch.float64, device=self.dev)
        ws = self._bm_ws
        _lib.check(self.lib.gee_bitmap_shard_encode(
            _device.ptr(r), _device.ptr(c), e, n, rb, re, k, flags,
            _device.ptr(deg_all) if deg_all is not None else None, _device.ptr(z), _device.ptr(ws), ws.numel(),
            _device.ptr(self._bm_err), _device.stream_handle()))
        if check:
            _lib.raise_device_errors(int(self._bm_err.item()), "sharded bitmap encode")
        return z


    # -- edge shuffle (distributed CSR build from edge-list slices) ----------
    def row_hist(self, rows, cols, n, directed):
        """Stream entries of this slice per coarse row bucket: int64[B]."""
        nb = int(self.lib.gee_shuffle_buckets(n))
        hist = torch.zeros(max(nb, 1), dtype=torch.int64, device=self.dev)
        _lib.check(self.lib.gee_shuffle_row_hist(_device.ptr(rows), _device.ptr(cols), int(rows.numel()), n,
                                                 int(bool(directed)), _device.ptr(hist), _device.stream_handle()))
        return hist[:nb]

    def shuffle_bounds(self, hist, n, world):
        """Row ranges with near-equal stream entries: int64[world + 1]."""
        bounds = torch.empty(world + 1, dtype=torch.int64, device=self.dev)
        _lib.check(self.lib.gee_shuffle_bounds(_device.ptr(hist), n, world, _device.ptr(bounds),
                                               _device.stream_handle()))
        return bounds

    def partition(self, rows, cols, w, directed, bounds, world):
        """Stable partition into [half][dest] send buckets; returns the three
        send buffers and the 2*world bucket sizes (host ints)."""
        e = int(rows.numel())
        cap = max(2 * e, 1)
        wt = _lib.W_UNIT if w is None else (_lib.W_F32 if w.dtype == torch.float32 else _lib.W_F64)
        out_r = torch.empty(cap, dtype=torch.int64, device=self.dev)
        out_c = torch.empty(cap, dtype=torch.int64, device=self.dev)
        out_w = None if w is None else torch.empty(cap, dtype=w.dtype, device=self.dev)
        counts = torch.empty(2 * world, dtype=torch.int64, device=self.dev)
        nb = _lib.size_query(self.lib.gee_partition_workspace, e, world)
        ws = _device.WORKSPACE.get(max(nb, 256), self.dev)
        _lib.check(self.lib.gee_partition(
            _device.ptr(rows), _device.ptr(cols), _device.ptr(w), wt, e, int(bool(directed)), _device.ptr(bounds),
            world, _device.ptr(out_r), _device.ptr(out_c), _device.ptr(out_w), _device.ptr(counts),
            _device.ptr(ws), ws.numel(), _device.stream_handle()))
        return out_r, out_c, out_w, counts.cpu().tolist()


# ---------------------------------------------------------------------------
# orchestration
# ---------------------------------------------------------------------------
def shard_plan(rows, cols, n, directed, world):
    return row_ranges(stream_row_counts(rows, cols, n, directed), world)


def encode_rows(ops, stream, labels, n, k, flags, ranges, rank, group=None):
    """Steps 2-5 for rank `rank` given its stream slice; returns Z[rb:re]."""
    rb, re = ranges[rank]
    r, c, w = stream
    y32_local, counts = ops.label_hist(labels[rb:re], k)
    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)        # class histogram
    y32 = all_gather_ranges(y32_local, ranges, group)                   # labels of every column
    inv = ops.inv_counts(counts)
    csr, scale = ops.csr_degree(r, c, w, n, flags)
    if flags & _lib.LAPLACIAN:
        scale = all_gather_ranges(scale[rb:re].contiguous(), ranges, group)  # degree scale vector
    return ops.embed(csr, rb, re, n, y32, inv, scale, k, flags)


def encode_rows_stream(ops, stream, labels, n, k, flags, ranges, rank, group=None, check=True, z=None):
    """Stream path for rank `rank` (unit or non-negative weights): partition
    its entries and compute its rows' degrees, ALL-GATHER of the degree
    vector (f64, N; Laplacian only -- labels are replicated, so n_k needs no
    collective), then the node table and Z[rb:re].  No host synchronisation
    unless `check`."""
    rb, re = ranges[rank]
    r, c, w = stream
    if getattr(ops, "_st", None) is None or ops._st["e"] != int(r.numel()) or ops._st["rb"] != rb:
        ops.st_prepare(r, c, w, n, rb, re, k, flags)
    deg_local = ops.st_degrees(r, c, w, labels)
    deg_all = all_gather_ranges(deg_local, ranges, group) if flags & _lib.LAPLACIAN else None
    z = ops.st_encode(deg_all, z)
    if check:
        ops.st_check()
    return z


def stream_ok(w) -> bool:
    """The stream path applies: unit weights, or weights all >= 0."""
    return w is None or bool((w >= 0).all())


def encode_rows_bitmap(ops, stream, labels, n, k, flags, ranges, rank, group=None, check=True):
    """Bitmap path for rank `rank` (unit weights): degrees of the local rows,
    ALL-GATHER of the degree vector (Laplacian only), then Z[rb:re]."""
    rb, re = ranges[rank]
    r, c, _ = stream
    deg_local = ops.bm_degrees(r, c, n, rb, re, labels, k, flags)
    deg_all = all_gather_ranges(deg_local, ranges, group) if flags & _lib.LAPLACIAN else None
    return ops.bm_encode(r, c, n, rb, re, k, flags, deg_all, check=check)


def encode_sharded(edges, labels, opts=None, group=None, ops=None):
    """Row-sharded encode of an EdgeList replicated on every rank.  Returns
    (z_local, (rb, re)): this rank's rows of Z."""
    from .graph import options_flags
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    ops = ops or GpuShardOps(_device.require_gpu())
    n, k = edges.n_nodes, labels.k_classes
    flags = options_flags(opts)
    ranges = shard_plan(edges.rows, edges.cols, n, edges.directed, world)
    rb, re = ranges[rank]
    dev = ops.dev
    e = edges.to_device(dev)
    _, w = e.weight_kind()
    stream = local_stream(e.rows, e.cols, w, edges.directed, rb, re)
    lab = _device.to_device(labels.labels, torch.int64, dev)
    nonneg = w is None or bool(e.nonneg)
    if ops.bitmap_ok(n, k, w is not None):
        z = encode_rows_bitmap(ops, stream, lab, n, k, flags, ranges, rank, group)
    elif nonneg and hasattr(ops, "st_prepare"):
        z = encode_rows_stream(ops, stream, lab, n, k, flags, ranges, rank, group)
    else:
        z = encode_rows(ops, stream, lab, n, k, flags, ranges, rank, group)
    return z, (rb, re)


# ---------------------------------------------------------------------------
# distributed CSR build: every rank starts from its own slice of the edge list
# ---------------------------------------------------------------------------
def shuffle_plan(ops, rows, cols, n, directed, world, group=None):
    """Row ranges from the ALL-REDUCED coarse row histogram of every rank's
    slice (device kernels; replaces the host stream_row_counts/row_ranges)."""
    hist = ops.row_hist(rows, cols, n, directed)
    dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=group)
    bounds = ops.shuffle_bounds(hist, n, world)
    b = bounds.cpu().tolist()
    return bounds, [(b[p], b[p + 1]) for p in range(world)]


def shuffle_stream(ops, rows, cols, w, directed, bounds, world, group=None):
    """ALL-TO-ALL of the stably partitioned slice: the originals region, then
    the mirrors region.  Concatenated in source-rank order they are this
    rank's slice of the symmetrised stream in stream order -- exactly what
    local_stream() selects from a replicated list (so the CSR is bitwise
    shard-invariant)."""
    out_r, out_c, out_w, counts = ops.partition(rows, cols, w, directed, bounds, world)
    send_o, send_m = counts[:world], counts[world:]
    dev = out_r.device
    sizes = torch.tensor([[send_o[d], send_m[d]] for d in range(world)], dtype=torch.int64, device=dev)
    got = torch.empty_like(sizes)
    dist.all_to_all_single(got.view(-1), sizes.view(-1), group=group)
    got = got.cpu().tolist()
    recv_o, recv_m = [g[0] for g in got], [g[1] for g in got]
    n_o = sum(send_o)

    def exchange(buf, lo, send, recv):
        out = torch.empty(sum(recv), dtype=buf.dtype, device=dev)
        dist.all_to_all_single(out, buf[lo:lo + sum(send)].contiguous(), recv, send, group=group)
        return out

    parts = []
    for buf in (out_r, out_c, out_w):
        if buf is None:
            parts.append(None)
            continue
        parts.append(torch.cat([exchange(buf, 0, send_o, recv_o), exchange(buf, n_o, send_m, recv_m)]))
    return parts[0], parts[1], parts[2]


def encode_distributed(rows, cols, weights, n, directed, labels, k, opts=None, group=None, ops=None):
    """Row-sharded encode from an edge list PARTITIONED across ranks: rank p
    passes its contiguous slice (rows, cols, weights: p-th stream range of the
    original EdgeList, slices in rank order) and the replicated labels.
    Device row histogram -> ALL-REDUCE -> row ranges -> stable partition ->
    ALL-TO-ALL edge shuffle -> encode_rows / encode_rows_bitmap.  Returns
    (z_local, (rb, re))."""
    from .errors import StructuralError
    from .graph import options_flags
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    ops = ops or GpuShardOps(_device.require_gpu())
    dev = ops.dev
    flags = options_flags(opts)
    rows = _device.to_device(rows, torch.int64, dev)
    cols = _device.to_device(cols, torch.int64, dev)
    if rows.numel() != cols.numel():
        raise StructuralError("rows and cols of the slice differ in length")
    if rows.numel():
        lo = torch.minimum(rows.min(), cols.min())
        hi = torch.maximum(rows.max(), cols.max())
        bad = torch.stack([lo < 0, hi >= n]).any().to(torch.int64)
    else:
        bad = torch.zeros((), dtype=torch.int64, device=dev)
    w = None
    unit = torch.ones((), dtype=torch.int64, device=dev)
    if weights is not None:
        w = weights if isinstance(weights, torch.Tensor) else torch.as_tensor(np.asarray(weights))
        w = w.to(dev)
        if w.dtype not in (torch.float32, torch.float64):
            w = w.to(torch.float64)
        if w.numel():
            bad = bad | (~torch.isfinite(w)).any().to(torch.int64)
            unit = (w == 1.0).all().to(torch.int64)
    flag = torch.stack([bad, 1 - unit])
    dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)   # any rank bad / any weight != 1.0
    flag = flag.cpu().tolist()
    if flag[0]:
        raise StructuralError("edge endpoints must lie in [0, n) and weights must be finite")
    if not flag[1]:
        w = None  # every weight is 1.0 on every rank: the unit-weight paths
    bounds, ranges = shuffle_plan(ops, rows, cols, n, directed, world, group)
    stream = shuffle_stream(ops, rows, cols, w, directed, bounds, world, group)
    lab = _device.to_device(labels.labels if hasattr(labels, "labels") else labels, torch.int64, dev)
    if ops.bitmap_ok(n, k, w is not None):
        z = encode_rows_bitmap(ops, stream, lab, n, k, flags, ranges, rank, group)
    else:
        z = encode_rows(ops, stream, lab, n, k, flags, ranges, rank, group)
    return z, ranges[rank]


def gather_z(z_local, ranges, group=None):
    """Row-sharded Z -> full Z on every rank (optional gather)."""
    k = z_local.shape[1]
    width = max(re - rb for rb, re in ranges)
    buf = torch.zeros((width, k), dtype=z_local.dtype, device=z_local.device)
    buf[: z_local.shape[0]] = z_local
    parts = [torch.empty_like(buf) for _ in ranges]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([parts[p][: re - rb] for p, (rb, re) in enumerate(ranges)])


# ---------------------------------------------------------------------------
# bench.py under torchrun
# ---------------------------------------------------------------------------
def bench_sharded(args, rank, world, dev):
    """Strong scaling of one config's step over `world` GPUs: every rank
    builds the same seeded input, keeps its stream slice (outside the timed
    region), then times label hist + collectives + CSR/degree + embed.
    value = input edges / max-over-ranks step time."""
    import json
    import statistics
    import sys

    sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
    from . import synth
    cfg = synth.make_config(args.config, device=dev)
    n, k, directed, flags = cfg["n"], cfg["k"], cfg["directed"], cfg["flags"]
    rows = torch.as_tensor(cfg["rows"], device=dev)
    cols = torch.as_tensor(cfg["cols"], device=dev)
    w = torch.as_tensor(cfg["weights"], device=dev)
    if bool((w == 1.0).all()):
        w = None
    lab = torch.as_tensor(cfg["labels"], device=dev)
    shuffle = bool(getattr(args, "shuffle", False))
    if shuffle:
        # distributed CSR build: this rank holds only its contiguous slice of
        # the original edge list; the whole shuffle is inside the timed region
        e_all = int(rows.numel())
        lo, hi = e_all * rank // world, e_all * (rank + 1) // world
        rs, cs = rows[lo:hi].clone(), cols[lo:hi].clone()
        ws_ = None if w is None else w[lo:hi].clone()
        del rows, cols, w
        ranges = None
    else:
        ranges = shard_plan(rows, cols, n, directed, world)
        rb, re = ranges[rank]
        stream = local_stream(rows, cols, w, directed, rb, re)
    ops = GpuShardOps(dev)
    from .graph import EmbedOptions
    opts = EmbedOptions(bool(flags & _lib.LAPLACIAN), bool(flags & _lib.DIAGONAL), bool(flags & _lib.CORRELATION))
    use_bm = (not shuffle) and ops.bitmap_ok(n, k, w is not None)
    if shuffle:
        def step():
            return encode_distributed(rs, cs, ws_, n, directed, lab, k, opts, ops=ops)
    elif use_bm:
        def step():
            return encode_rows_bitmap(ops, stream, lab, n, k, flags, ranges, rank, check=False)
    else:
        def step():
            return encode_rows(ops, stream, lab, n, k, flags, ranges, rank)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    run = step
    graphed = False
    if use_bm and not args.eager:
        # the whole step (kernels + the NCCL all-gather) as one CUDA graph
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step()
            run = g.replay
            graphed = True
            run()
            torch.cuda.synchronize()
        except Exception as ex:  # capture unsupported here: time eager launches
            print(f"[rank {rank}] CUDA graph capture failed ({ex}); timing eager launches", file=sys.stderr)
            run = step
    if use_bm:
        _lib.raise_device_errors(int(ops._bm_err.item()), "sharded bitmap encode")
    times = []
    for _ in range(args.steps):
        dist.barrier()
        torch.cuda.synchronize()
        s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        run()
        t.record()
        torch.cuda.synchronize()
        dist.barrier()
        times.append(s.elapsed_time(t))
    ms = torch.tensor([statistics.mean(times)], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        e = int(cfg["e"])
        line = {"metric": "GEE edges/sec", "value": e / (float(ms) * 1e-3), "unit": "edges/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(ms),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded, BASELINE.json shapes)",
                "config": {"workload": f"configs[{args.config}] {cfg['name']}", "n_nodes": n, "n_edges": e,
                           "k_classes": k,
                           "parallelism": (f"edge-list slices x{world}: device row histogram, NCCL all-reduce, "
                                           "stable partition, NCCL all-to-all edge shuffle, then the row-sharded "
                                           "encode" if shuffle else
                                           f"row-sharded x{world}, bitmap path (NCCL all-gather of degrees)"
                                           if use_bm else f"row-sharded x{world} (NCCL all-reduce n_k, "
                                           "all-gather labels + Laplacian scale)"),
                           "cuda_graph": graphed}}
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0
