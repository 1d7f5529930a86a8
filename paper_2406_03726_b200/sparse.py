"""Device-resident CSR and the reference's sparse-core operations on it.

Mirrors pkg/src/graphee/sparse.py (CsrMatrix :19-114, add_identity :184-190,
degree_vector :193-196, laplacian_normalize :199-226) and the kernel seam
_kernels.coo_to_csr (:39-130).  Storage on the B200: index_pointers int64,
col_indices int32 (node ids < 2^31), data float64 -- 12 bytes per stored
entry instead of the reference's 16.  ``to_numpy()`` returns the reference's
exact arrays (int64 / int64 / float64), bit for bit.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device, _lib
from .errors import NumericalDomainError, StructuralError


class CsrMatrix:
    """Immutable sparse matrix in compressed sparse row form, on a CUDA device."""

    def __init__(self, n_rows: int, n_cols: int, index_pointers: torch.Tensor,
                 col_indices: torch.Tensor, data: torch.Tensor):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        # device storage (row_ptr int64, col int32, val float64); the
        # reference-named fields below are host views with the reference's
        # dtypes (sparse.py:20-27: int64 / int64 / float64 numpy arrays)
        self.row_ptr_d = index_pointers
        self.col_d = col_indices
        self.val_d = data
        self._host = None

    def _numpy(self):
        if self._host is None:
            self._host = (self.row_ptr_d.cpu().numpy().astype(np.int64, copy=False),
                          self.col_d.cpu().numpy().astype(np.int64),
                          self.val_d.cpu().numpy())
            for a in self._host:
                a.flags.writeable = False
        return self._host

    @property
    def index_pointers(self) -> np.ndarray:
        return self._numpy()[0]

    @property
    def col_indices(self) -> np.ndarray:
        return self._numpy()[1]

    @property
    def data(self) -> np.ndarray:
        return self._numpy()[2]

    # ---- construction ------------------------------------------------------
    @classmethod
    def from_host(cls, n_rows, n_cols, index_pointers, col_indices, data, device=None):
        dev = torch.device(device) if device is not None else _device.require_gpu()
        return cls(n_rows, n_cols, _device.to_device(index_pointers, torch.int64, dev),
                   _device.to_device(col_indices, torch.int32, dev),
                   _device.to_device(data, torch.float64, dev))

    @classmethod
    def coerce(cls, m, device=None) -> "CsrMatrix":
        """Accept this class or any CsrMatrix-like object (e.g. the reference's)."""
        if isinstance(m, CsrMatrix):
            return m
        return cls.from_host(m.n_rows, m.n_cols, m.index_pointers, m.col_indices, m.data, device)

    @classmethod
    def from_edges(cls, edges) -> "CsrMatrix":
        """EdgeList.to_csr() on the device (graph_io.py:78-92 + _kernels.py:73-130)."""
        dev = _device.require_gpu()
        e = edges.to_device(dev)
        return _build(e.rows, e.cols, e.weight_kind(), e.n_edges, e.n_nodes, e.n_nodes,
                      e.directed, dev)

    @classmethod
    def from_triplets(cls, rows, cols, vals, n_rows: int, n_cols: int, check: bool = True):
        """sparse.py:33-68: duplicates summed in input order, exact zeros dropped."""
        rows = np.ascontiguousarray(rows, dtype=np.int64) if not isinstance(rows, torch.Tensor) else rows
        cols = np.ascontiguousarray(cols, dtype=np.int64) if not isinstance(cols, torch.Tensor) else cols
        vals = np.ascontiguousarray(vals, dtype=np.float64) if not isinstance(vals, torch.Tensor) else vals
        if not (rows.shape == cols.shape == vals.shape):
            raise StructuralError("triplet arrays must have equal length")
        if n_rows < 0 or n_cols < 0:
            raise StructuralError("matrix shape must be non-negative")
        if check and rows.shape[0] and isinstance(rows, np.ndarray):
            bad = (rows < 0) | (rows >= n_rows) | (cols < 0) | (cols >= n_cols)
            if bad.any():
                e = int(np.flatnonzero(bad)[0])
                raise StructuralError(
                    f"triplet ({rows[e]}, {cols[e]}, {vals[e]}) outside {n_rows}x{n_cols} matrix")
            finite = np.isfinite(vals)
            if not finite.all():
                e = int(np.flatnonzero(~finite)[0])
                raise StructuralError(
                    f"triplet ({rows[e]}, {cols[e]}, {vals[e]}) has a non-finite value")
        dev = _device.require_gpu()
        r = _device.to_device(rows, torch.int64, dev)
        c = _device.to_device(cols, torch.int64, dev)
        v = _device.to_device(vals, torch.float64, dev)
        if check and r.shape[0] and not isinstance(rows, np.ndarray):
            # device inputs get the same checks, on the device (one host sync)
            bad = (r < 0) | (r >= n_rows) | (c < 0) | (c >= n_cols)
            nonfin = ~torch.isfinite(v)
            flags = torch.stack([bad.any(), nonfin.any()]).cpu()
            if bool(flags[0]):
                e = int(torch.nonzero(bad)[0])
                raise StructuralError(
                    f"triplet ({int(r[e])}, {int(c[e])}, {float(v[e])}) outside {n_rows}x{n_cols} matrix")
            if bool(flags[1]):
                e = int(torch.nonzero(nonfin)[0])
                raise StructuralError(
                    f"triplet ({int(r[e])}, {int(c[e])}, {float(v[e])}) has a non-finite value")
        return _build(r, c, (_lib.W_F64, v), int(r.shape[0]), n_rows, n_cols, True, dev)

    # ---- accessors -----------------------------------------------------------
    @property
    def nnz(self) -> int:
        return int(self.val_d.shape[0])

    @property
    def device(self) -> torch.device:
        return self.val_d.device

    def to_numpy(self):
        """(index_pointers int64, col_indices int64, data float64) on the host."""
        return self._numpy()

    def row_ids(self) -> np.ndarray:
        ip = self.index_pointers
        return np.repeat(np.arange(self.n_rows, dtype=np.int64), np.diff(ip))

    def row(self, r: int):
        if not 0 <= r < self.n_rows:
            raise IndexError(f"row {r} out of range for {self.n_rows} rows")
        lo, hi = (int(x) for x in self.index_pointers[r:r + 2])
        return self.col_indices[lo:hi], self.data[lo:hi]

    def to_triplets(self):
        return self.row_ids(), self.col_indices.copy(), self.data.copy()

    def to_dense(self) -> np.ndarray:
        ip, c, d = self.to_numpy()
        dense = np.zeros((self.n_rows, self.n_cols))
        if d.size:
            dense[np.repeat(np.arange(self.n_rows), np.diff(ip)), c] = d
        return dense

    def validate(self) -> None:
        """Every structural invariant of sparse.py:93-114; StructuralError if broken."""
        ptr, cols, data = self.to_numpy()
        if ptr.shape[0] != self.n_rows + 1:
            raise StructuralError("index_pointers length must be n_rows + 1")
        if ptr[0] != 0 or ptr[-1] != data.shape[0]:
            raise StructuralError("index_pointers must start at 0 and end at nnz")
        if np.any(np.diff(ptr) < 0):
            raise StructuralError("index_pointers must be non-decreasing")
        if cols.shape[0] != data.shape[0]:
            raise StructuralError("col_indices and data must have equal length")
        if data.size:
            if cols.min() < 0 or cols.max() >= self.n_cols:
                raise StructuralError("column index out of range")
            rid = np.repeat(np.arange(self.n_rows, dtype=np.int64), np.diff(ptr))
            same = rid[1:] == rid[:-1]
            if not np.all(cols[1:][same] > cols[:-1][same]):
                raise StructuralError("columns must be strictly increasing within rows")
            if np.any(data == 0.0):
                raise StructuralError("stored values must not be exactly zero")
            if not np.isfinite(data).all():
                raise StructuralError("stored values must be finite")


def _build(rows, cols, weight_kind, n_edges, n_rows, n_cols, directed, dev) -> CsrMatrix:
    lib = _lib.load()
    wt, w = weight_kind
    cap = max(n_edges if directed else 2 * n_edges, 1)
    row_ptr = torch.empty(n_rows + 1, dtype=torch.int64, device=dev)
    col = torch.empty(cap, dtype=torch.int32, device=dev)
    val = torch.empty(cap, dtype=torch.float64, device=dev)
    nnz = torch.zeros(1, dtype=torch.int64, device=dev)
    err = _device.error_word(dev)
    with torch.cuda.device(dev):
        nb = _lib.size_query(lib.gee_csr_build_workspace, n_edges, n_rows, n_cols, int(directed))
        ws = _device.WORKSPACE.get(nb, dev)
        _lib.check(lib.gee_csr_build(
            _device.ptr(rows), _device.ptr(cols), _device.ptr(w), wt, n_edges, n_rows, n_cols,
            int(directed), 1, _device.ptr(row_ptr), None, _device.ptr(col), _device.ptr(val),
            _device.ptr(nnz), 0, None, None, _device.ptr(ws), ws.numel(), _device.ptr(err),
            _device.stream_handle()))
    _device.check_device_errors(err, "to_csr")
    k = int(nnz.item())
    return CsrMatrix(n_rows, n_cols, row_ptr, col[:k], val[:k])


def _require_square(a: CsrMatrix, what: str) -> None:
    if a.n_rows != a.n_cols:
        raise StructuralError(f"{what} requires a square matrix, got {a.n_rows}x{a.n_cols}")


def add_identity(a) -> CsrMatrix:
    """Return A + I (sparse.py:184-190; _kernels.py:169-198), bit-exact."""
    a = CsrMatrix.coerce(a)
    _require_square(a, "add_identity")
    lib = _lib.load()
    dev = a.device
    n = a.n_rows
    out_ptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    cap = max(a.nnz + n, 1)
    out_col = torch.empty(cap, dtype=torch.int32, device=dev)
    out_val = torch.empty(cap, dtype=torch.float64, device=dev)
    nnz = torch.zeros(1, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        nb = _lib.size_query(lib.gee_add_identity_workspace, n)
        ws = _device.WORKSPACE.get(nb, dev)
        _lib.check(lib.gee_add_identity(
            _device.ptr(a.row_ptr_d), _device.ptr(a.col_d), _device.ptr(a.val_d), n,
            _device.ptr(out_ptr), _device.ptr(out_col), _device.ptr(out_val), _device.ptr(nnz),
            _device.ptr(ws), ws.numel(), _device.stream_handle()))
    k = int(nnz.item())
    return CsrMatrix(n, n, out_ptr, out_col[:k], out_val[:k])


def degree_vector(a, diagonal: bool = False, with_scale: bool = False):
    """Weighted degree per row (sparse.py:193-196) -- of A, or of A+I when
    `diagonal` (the encode path fuses the identity instead of building it).
    Bit-exact with np.bincount's storage-order fold.  Returns a device
    float64 tensor (and the Laplacian scale 1/sqrt(d) when `with_scale`)."""
    a = CsrMatrix.coerce(a)
    _require_square(a, "degree_vector")
    lib = _lib.load()
    dev = a.device
    n = a.n_rows
    deg = torch.empty(n, dtype=torch.float64, device=dev)
    scale = torch.empty(n, dtype=torch.float64, device=dev) if with_scale else None
    err = _device.error_word(dev)
    with torch.cuda.device(dev):
        _lib.check(lib.gee_degree(
            _device.ptr(a.row_ptr_d), _device.ptr(a.col_d), _device.ptr(a.val_d), n,
            _lib.DIAGONAL if diagonal else 0, _device.ptr(deg), _device.ptr(scale),
            _device.ptr(err), _device.stream_handle()))
    if with_scale:
        _device.check_device_errors(err, "degree_vector")
        return deg, scale
    return deg


def laplacian_normalize(a, degrees) -> CsrMatrix:
    """e_ij -> (e_ij * s_i) * s_j, s = d^-1/2 (0 where d == 0), zeros pruned
    (sparse.py:199-226), bit-exact."""
    a = CsrMatrix.coerce(a)
    _require_square(a, "laplacian_normalize")
    dev = a.device
    deg = _device.to_device(degrees, torch.float64, dev)
    if deg.shape[0] != a.n_rows:
        raise StructuralError(f"degree vector length {deg.shape[0]} != matrix size {a.n_rows}")
    lib = _lib.load()
    n = a.n_rows
    out_ptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    cap = max(a.nnz, 1)
    out_col = torch.empty(cap, dtype=torch.int32, device=dev)
    out_val = torch.empty(cap, dtype=torch.float64, device=dev)
    nnz = torch.zeros(1, dtype=torch.int64, device=dev)
    err = _device.error_word(dev)
    with torch.cuda.device(dev):
        nb = _lib.size_query(lib.gee_laplacian_normalize_workspace, n)
        ws = _device.WORKSPACE.get(nb, dev)
        _lib.check(lib.gee_laplacian_normalize(
            _device.ptr(a.row_ptr_d), _device.ptr(a.col_d), _device.ptr(a.val_d), n,
            _device.ptr(deg), _device.ptr(out_ptr), _device.ptr(out_col), _device.ptr(out_val),
            _device.ptr(nnz), _device.ptr(ws), ws.numel(), _device.ptr(err),
            _device.stream_handle()))
    bits = int(err.item())
    if bits & _lib.ERR_NEG_DEGREE:
        raise NumericalDomainError("negative degree under Laplacian normalization")
    k = int(nnz.item())
    return CsrMatrix(n, n, out_ptr, out_col[:k], out_val[:k])
