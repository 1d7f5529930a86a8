"""encode(): the reference's public entry point, on the B200.

Reference: pkg/src/graphee/embedding.py:110-131 (``encode``), called as
``encode(EdgeList(...).to_csr(), labels, opts)`` (cli.py:108-109, :176).
Both call forms are accepted:

* an EdgeList (ours or the reference's)  -> the fused device pipeline
  gee_encode_edges: K1 label histogram, K2 CSR assembly with the K3 degree
  fused in, K4 embedding with Laplacian/diagonal in its load path and
  correlation in its epilogue -- the whole reference timed region;
* a CsrMatrix (ours, or any object with the reference's CsrMatrix fields)
  -> gee_degree (if Laplacian) + gee_embed.

Errors follow the reference: StructuralError for shape/label problems
(embedding.py:115-122), NumericalDomainError for negative degrees
(sparse.py:211-212) and non-finite rows under correlation
(embedding.py:137-138).  The result is a float64 (N, K) numpy array (the
drop-in contract) or, with ``out="torch"``, the device tensor.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device, _lib
from .errors import NumericalDomainError, StructuralError
from .graph import EdgeList, EmbedOptions, LabelVector, options_flags
from .sparse import CsrMatrix


def _labels_of(labels):
    if isinstance(labels, LabelVector):
        return labels
    return LabelVector(labels.labels, labels.k_classes)


def _edges_of(edges):
    if isinstance(edges, EdgeList):
        return edges
    # a duck-typed (e.g. the reference's) EdgeList: the reference validated it
    # at construction (graph_io.py:58-72); weights are only checked for sign
    out = EdgeList(edges.n_nodes, edges.rows, edges.cols, edges.weights, edges.directed, validate=False)
    w = out.weights
    if w is not None and out.n_edges:
        if isinstance(w, np.ndarray):
            out.unit_weights = bool((w == 1.0).all())
            out.nonneg = bool((w >= 0).all())
        else:
            f = torch.stack([(w == 1.0).all(), (w >= 0).all()]).cpu()
            out.unit_weights, out.nonneg = bool(f[0]), bool(f[1])
    return out


def label_tables(labels, device=None):
    """K1: (y32 int32[N], counts int64[K], inv_nk float64[K]) on the device."""
    labels = _labels_of(labels)
    dev = torch.device(device) if device is not None else _device.require_gpu()
    lab = _device.to_device(labels.labels, torch.int64, dev)
    n, k = len(labels), labels.k_classes
    y32 = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    counts = torch.empty(k, dtype=torch.int64, device=dev)
    inv = torch.empty(k, dtype=torch.float64, device=dev)
    err = _device.error_word(dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.load().gee_label_hist(_device.ptr(lab), n, k, _device.ptr(y32),
                                              _device.ptr(counts), _device.ptr(inv),
                                              _device.ptr(err), _device.stream_handle()))
    _device.check_device_errors(err, "labels")
    return y32[:n], counts, inv


class GeeEncoder:
    """Reusable plan for repeated edge-list -> Z calls of one shape.

    Holds the workspace, the error word and the output; ``run`` launches the
    fused pipeline on the current stream without synchronising (check=False)
    so a caller can time or graph-capture it.  ``nonneg=True`` asserts every
    weight is >= 0 (EdgeList.nonneg), which enables the bucketed stream path;
    ``dtype=torch.float32`` produces Z in float32 (north_star's optional fp32
    path: f64 accumulation, f32 storage, 1e-5).
    """

    def __init__(self, n_nodes: int, n_edges: int, k_classes: int, directed: bool,
                 opts: EmbedOptions | None = None, device=None, *, nonneg: bool = False,
                 dtype: torch.dtype = torch.float64):
        self.dev = torch.device(device) if device is not None else _device.require_gpu()
        self.n, self.e, self.k = int(n_nodes), int(n_edges), int(k_classes)
        self.directed = bool(directed)
        self.flags = options_flags(opts)
        self.nonneg = bool(nonneg)
        if dtype not in (torch.float64, torch.float32):
            raise ValueError("dtype must be torch.float64 or torch.float32")
        self.dtype = dtype
        lib = _lib.load()
        with torch.cuda.device(self.dev):
            # the assembly path (and its workspace) depends on the weight kind
            nb = max(_lib.size_query(lib.gee_encode_edges_workspace, self.e, self.n, self.k,
                                     int(self.directed), wt) for wt in (_lib.W_UNIT, _lib.W_F64))
        self.ws = torch.empty(max(nb, 256), dtype=torch.uint8, device=self.dev)
        self.z = torch.empty((self.n, self.k), dtype=dtype, device=self.dev)
        self.err = _device.error_word(self.dev)

    def run_flags(self, weights) -> int:
        f = self.flags
        if self.nonneg or weights is None:
            f |= _lib.NONNEG
        if self.dtype == torch.float32:
            f |= _lib.FP32
        return f

    def run(self, rows, cols, weights, labels, *, check: bool = True, out=None) -> torch.Tensor:
        """rows/cols int64, weights float64/float32/None, labels int64 -- device tensors."""
        if weights is None:
            wt = _lib.W_UNIT
        else:
            wt = _lib.W_F32 if weights.dtype == torch.float32 else _lib.W_F64
        z = self.z if out is None else out
        if check:
            self.err.zero_()
        flags = self.run_flags(weights)
        st = _lib.load().gee_encode_edges(
            _device.ptr(rows), _device.ptr(cols), _device.ptr(weights), wt, self.e, self.n,
            int(self.directed), _device.ptr(labels), self.k, flags, _device.ptr(z),
            _device.ptr(self.ws), self.ws.numel(), _device.ptr(self.err), _device.stream_handle())
        if st == _lib.GEE_E_ARG and self.dtype == torch.float32 and not (flags & _lib.NONNEG):
            # float32 Z comes from the stream path; signed weights take the exact
            # f64 CSR path and are narrowed once
            z64 = torch.empty((self.n, self.k), dtype=torch.float64, device=self.dev)
            _lib.check(_lib.load().gee_encode_edges(
                _device.ptr(rows), _device.ptr(cols), _device.ptr(weights), wt, self.e, self.n,
                int(self.directed), _device.ptr(labels), self.k, flags & ~_lib.FP32, _device.ptr(z64),
                _device.ptr(self.ws), self.ws.numel(), _device.ptr(self.err), _device.stream_handle()))
            z.copy_(z64)
        else:
            _lib.check(st)
        if check:
            bits = int(self.err.item())
            if bits & _lib.ERR_NEG_WEIGHT and self.nonneg:
                # the non-negativity assertion was wrong: recompute on the exact path
                self.nonneg = False
                return self.run(rows, cols, weights, labels, check=True, out=out)
            _lib.raise_device_errors(bits, "encode")
        return z

    def capture(self, rows, cols, weights, labels, *, profile: bool = False):
        """Capture the pipeline for these device inputs into a CUDA graph
        (removes host launch gaps between the ~12 kernels).  With `profile`,
        per-kernel event-record nodes are captured too (gee_profile_read
        reports per-kernel times after each replay)."""
        lib = _lib.load()
        self.run(rows, cols, weights, labels, check=True)  # warm-up: attributes, errors
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            if profile:
                lib.gee_profile_start(torch.cuda.current_stream().cuda_stream)
            self.run(rows, cols, weights, labels, check=False)
            if profile:
                lib.gee_profile_stop()
        torch.cuda.synchronize()
        return self.graph

    def replay(self) -> torch.Tensor:
        self.graph.replay()
        return self.z

    def attach_host(self, rows, cols, weights, labels, *, depth: int = 2):
        """Register host inputs for run_host() / run_host_async(): pinned
        staging copies, `depth` sets of device input buffers and outputs, and
        pinned host outputs.  Returns (h2d_bytes, d2h_bytes) per run."""
        def pin(a):
            t = torch.from_numpy(np.ascontiguousarray(a)) if isinstance(a, np.ndarray) else a.cpu()
            return t.pin_memory()
        self._h = [pin(rows), pin(cols), None if weights is None else pin(weights), pin(labels)]
        self._depth = max(1, int(depth))
        self._d = [[None if h is None else torch.empty_like(h, device=self.dev) for h in self._h]
                   for _ in range(self._depth)]
        self._zd = [self.z] + [torch.empty_like(self.z) for _ in range(self._depth - 1)]
        self._zhs = [torch.empty((self.n, self.k), dtype=self.dtype).pin_memory() for _ in range(self._depth)]
        self._zh = self._zhs[0]
        self._s_in = torch.cuda.Stream(self.dev)
        self._s_out = torch.cuda.Stream(self.dev)
        mk = lambda: [torch.cuda.Event() for _ in range(self._depth)]  # noqa: E731
        self._ev_in_free, self._ev_h2d, self._ev_comp, self._ev_out_free = mk(), mk(), mk(), mk()
        self._step = 0
        h2d = sum(h.numel() * h.element_size() for h in self._h if h is not None)
        return h2d, self._zh.numel() * self._zh.element_size()

    def run_host(self, *, check: bool = True) -> torch.Tensor:
        """Host -> device copies, the fused pipeline, device -> host Z; all
        stream-ordered on the current stream (the synchronous end-to-end call)."""
        d = self._d[0]
        for h, x in zip(self._h, d):
            if h is not None:
                x.copy_(h, non_blocking=True)
        rows, cols, w, lab = d
        z = self.run(rows, cols, w, lab, check=False)
        self._zh.copy_(z, non_blocking=True)
        if check:
            torch.cuda.current_stream().synchronize()
            _device.check_device_errors(self.err, "encode")
        return self._zh

    def run_host_async(self):
        """One end-to-end step for a stream of encodes: its inputs go up on a
        copy stream while the previous step computes, its Z comes down on a
        second copy stream while the next step's inputs go up (PCIe is full
        duplex).  Buffers rotate over `depth` slots.  Returns (host Z, event):
        the host Z is valid once the event has completed."""
        b = self._step % self._depth
        self._step += 1
        cs = torch.cuda.current_stream(self.dev)
        with torch.cuda.stream(self._s_in):
            self._s_in.wait_event(self._ev_in_free[b])  # the previous compute on slot b read its inputs
            for h, x in zip(self._h, self._d[b]):
                if h is not None:
                    x.copy_(h, non_blocking=True)
            self._ev_h2d[b].record(self._s_in)
        cs.wait_event(self._ev_h2d[b])
        cs.wait_event(self._ev_out_free[b])  # slot b's previous Z has reached the host
        rows, cols, w, lab = self._d[b]
        self.run(rows, cols, w, lab, check=False, out=self._zd[b])
        self._ev_in_free[b].record(cs)
        self._ev_comp[b].record(cs)
        with torch.cuda.stream(self._s_out):
            self._s_out.wait_event(self._ev_comp[b])
            self._zhs[b].copy_(self._zd[b], non_blocking=True)
            self._ev_out_free[b].record(self._s_out)
        return self._zhs[b], self._ev_out_free[b]


def _check_shapes(n_rows, n_cols, labels):
    if n_rows != n_cols:
        raise StructuralError(f"adjacency must be square, got {n_rows}x{n_cols}")
    if len(labels) != n_rows:
        raise StructuralError(f"label count {len(labels)} != node count {n_rows}")


_ENCODERS: dict = {}
_ENCODER_CACHE = 4


def _encoder(n, e, k, directed, flags, nonneg, dtype, dev) -> GeeEncoder:
    """Per-shape plan cache (workspace + output reused across calls)."""
    key = (dev, n, e, k, directed, flags, nonneg, dtype)
    enc = _ENCODERS.pop(key, None)
    if enc is None:
        while len(_ENCODERS) >= _ENCODER_CACHE:
            _ENCODERS.pop(next(iter(_ENCODERS)))
        enc = GeeEncoder(n, e, k, directed, None, dev, nonneg=nonneg, dtype=dtype)
        enc.flags = flags
    _ENCODERS[key] = enc  # most recently used last
    return enc


def encode(adj, labels, opts=None, *, out: str = "numpy", dtype=torch.float64):
    """Embed via the sparse pipeline on the GPU; returns a dense (N, K) array
    (float64, or float32 with dtype=torch.float32 -- the optional fp32 path)."""
    labels = _labels_of(labels)
    flags = options_flags(opts)
    dev = _device.require_gpu()
    # (a CsrMatrix's reference-named fields are host copies: never touch them here)
    if isinstance(adj, CsrMatrix) or (not isinstance(adj, EdgeList) and hasattr(adj, "index_pointers")):
        z = _encode_csr(CsrMatrix.coerce(adj, dev), labels, flags, dev)
        if dtype == torch.float32:
            z = z.to(torch.float32)
    else:
        edges = _edges_of(adj)
        _check_shapes(edges.n_nodes, edges.n_nodes, labels)
        e = edges.to_device(dev)
        lab = _device.to_device(labels.labels, torch.int64, dev)
        wt_code, w = e.weight_kind()
        enc = _encoder(e.n_nodes, e.n_edges, labels.k_classes, e.directed, flags, bool(e.nonneg), dtype, dev)
        z = enc.run(e.rows, e.cols, w, lab, check=True)
        if out == "torch":
            z = z.clone()  # the plan's output buffer is reused by the next call
    if out == "torch":
        return z
    return z.cpu().numpy()


def _encode_csr(a: CsrMatrix, labels: LabelVector, flags: int, dev) -> torch.Tensor:
    _check_shapes(a.n_rows, a.n_cols, labels)
    lib = _lib.load()
    n, k = a.n_rows, labels.k_classes
    y32, _, inv = label_tables(labels, dev)
    err = _device.error_word(dev)
    scale = None
    with torch.cuda.device(dev):
        if flags & _lib.LAPLACIAN:
            deg = torch.empty(n, dtype=torch.float64, device=dev)
            scale = torch.empty(n, dtype=torch.float64, device=dev)
            _lib.check(lib.gee_degree(
                _device.ptr(a.row_ptr_d), _device.ptr(a.col_d), _device.ptr(a.val_d), n,
                flags & _lib.DIAGONAL, _device.ptr(deg), _device.ptr(scale), _device.ptr(err),
                _device.stream_handle()))
        z = torch.empty((n, k), dtype=torch.float64, device=dev)
        nb = _lib.size_query(lib.gee_embed_workspace, n, n)
        ws = _device.WORKSPACE.get(nb, dev)
        _lib.check(lib.gee_embed(
            _device.ptr(a.row_ptr_d), None, _device.ptr(a.col_d), _device.ptr(a.val_d), 0,
            n, n, _device.ptr(y32), _device.ptr(inv), _device.ptr(scale), k, flags, _device.ptr(z), k,
            _device.ptr(ws), ws.numel(), _device.ptr(err), _device.stream_handle()))
    _device.check_device_errors(err, "encode")
    return z


def build_weight_matrix(labels):
    """W as the reference builds it (embedding.py:92-107), materialised on the
    device by gee_weight_matrix as an N x K CsrMatrix: row j holds 1/n_{Y_j}
    at column Y_j, unlabeled rows are empty.  The encode path never needs it
    (gee_embed reads y32 + 1/n_k instead)."""
    labels = _labels_of(labels)
    if labels.k_classes < 1:
        raise StructuralError("k_classes must be at least 1")
    y32, _, inv = label_tables(labels)
    dev = y32.device
    n = len(labels)
    lib = _lib.load()
    ptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    cols = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    vals = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        ws = _device.WORKSPACE.get(_lib.size_query(lib.gee_weight_matrix_workspace, n), dev)
        _lib.check(lib.gee_weight_matrix(_device.ptr(y32), n, _device.ptr(inv), _device.ptr(ptr),
                                         _device.ptr(cols), _device.ptr(vals), _device.ptr(ws), ws.numel(),
                                         _device.stream_handle()))
    nnz = int(ptr[n].item())
    return CsrMatrix(n, labels.k_classes, ptr, cols[:nnz], vals[:nnz])


def encode_reference(edges, labels, opts=None, *, out: str = "numpy"):
    """The reference's edge-stream embedding (embedding.py:146-200): Z from
    the (i, j, e_ij) triplets with the options applied as edge-level
    transforms, no CSR.  On the B200 this is the same device pipeline as
    encode(EdgeList) -- the bucketed stream encode accumulates straight off
    the triplet stream exactly as the reference's bincount does, up to the
    summation order (results within 1e-12).  Reference
    semantics kept: only the label count is checked (no squareness check,
    embedding.py:158-159), and under correlation a non-finite Z is NOT an
    error -- rows are divided by sqrt(sum z*z) as numpy would
    (embedding.py:195-199), NaN/inf propagating."""
    opts = EmbedOptions() if opts is None else opts
    labels = _labels_of(labels)
    e = _edges_of(edges)
    if len(labels) != e.n_nodes:
        raise StructuralError(f"label count {len(labels)} != node count {e.n_nodes}")
    try:
        z = encode(e, labels, opts, out="torch")
    except NumericalDomainError as exc:
        if "non-finite" not in str(exc) or not opts.correlation:
            raise
        z = encode(e, labels, EmbedOptions(opts.laplacian, opts.diagonal, False), out="torch")
        norms = torch.sqrt((z * z).sum(dim=1))
        nz = norms > 0
        z[nz] = z[nz] / norms[nz, None]
    return z if out == "torch" else z.cpu().numpy()


def spmm_weight(a, labels, opts=None, *, out: str = "numpy"):
    """spmm(A, build_weight_matrix(labels)).to_dense() without building W."""
    a = CsrMatrix.coerce(a)
    return encode(a, labels, EmbedOptions() if opts is None else opts, out=out)
