"""ctypes wrapper over oracle/libgee_oracle.so -- TEST INFRASTRUCTURE ONLY.

The CPU restatement of the reference `graphee` sparse-GEE path
(pkg/src/graphee/{graph_io,sparse,_kernels,embedding}.py).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this module; the product package never does.

Pinned against the reference itself: tests/test_oracle_golden.py compares
every function here with fixtures that tests/golden/make_golden.py generated
by importing the reference package in the build container.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libgee_oracle.so")

LAPLACIAN = 1
DIAGONAL = 2
CORRELATION = 4

OK = 0
E_NEG_DEGREE = 2
E_NONFINITE = 3

_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)


def build() -> str:
    """Compile libgee_oracle.so with the committed Makefile (gcc only)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.gor_symmetrize.restype = ctypes.c_int64
        L.gor_symmetrize.argtypes = [_i64p, _i64p, _f64p, ctypes.c_int64, ctypes.c_int,
                                     _i64p, _i64p, _f64p]
        L.gor_coo_to_csr.restype = ctypes.c_int64
        L.gor_coo_to_csr.argtypes = [_i64p, _i64p, _f64p, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_int64, _i64p, _i64p, _f64p]
        L.gor_add_identity.restype = ctypes.c_int64
        L.gor_add_identity.argtypes = [_i64p, _i64p, _f64p, ctypes.c_int64, _i64p, _i64p, _f64p]
        L.gor_degree.restype = None
        L.gor_degree.argtypes = [_i64p, _f64p, ctypes.c_int64, _f64p]
        L.gor_laplacian_normalize.restype = ctypes.c_int
        L.gor_laplacian_normalize.argtypes = [_i64p, _i64p, _f64p, ctypes.c_int64, _f64p,
                                              _i64p, _i64p, _f64p, _i64p]
        L.gor_class_counts.restype = None
        L.gor_class_counts.argtypes = [_i64p, ctypes.c_int64, ctypes.c_int64, _i64p]
        L.gor_spmm_onehot_dense.restype = None
        L.gor_spmm_onehot_dense.argtypes = [_i64p, _i64p, _f64p, ctypes.c_int64, _i64p, _i64p,
                                            ctypes.c_int64, _f64p]
        L.gor_correlate_rows.restype = ctypes.c_int
        L.gor_correlate_rows.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int64]
        L.gor_encode_edges.restype = ctypes.c_int
        L.gor_encode_edges.argtypes = [_i64p, _i64p, _f64p, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_int, _i64p, ctypes.c_int64, ctypes.c_uint,
                                       _f64p, _i64p, _i64p, _f64p, _i64p, _f64p]
        _lib = L
    return _lib


def _p64(a):
    return a.ctypes.data_as(_i64p)


def _pf(a):
    return a.ctypes.data_as(_f64p)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def symmetrize(rows, cols, w, directed: bool):
    """graph_io.py:78-92 concatenation order."""
    rows, cols, w = _i64(rows), _i64(cols), _f64(w)
    e = rows.size
    cap = max(2 * e, 1)
    r = np.empty(cap, np.int64)
    c = np.empty(cap, np.int64)
    v = np.empty(cap, np.float64)
    m = lib().gor_symmetrize(_p64(rows), _p64(cols), _pf(w), e, int(directed),
                             _p64(r), _p64(c), _pf(v))
    return r[:m].copy(), c[:m].copy(), v[:m].copy()


def coo_to_csr(rows, cols, vals, n_rows: int, n_cols: int):
    """_kernels.py:73-130 (bitwise twin of the reference numba kernel)."""
    rows, cols, vals = _i64(rows), _i64(cols), _f64(vals)
    m = rows.size
    indptr = np.zeros(n_rows + 1, np.int64)
    oc = np.empty(max(m, 1), np.int64)
    ov = np.empty(max(m, 1), np.float64)
    nnz = lib().gor_coo_to_csr(_p64(rows), _p64(cols), _pf(vals), m, n_rows, n_cols,
                               _p64(indptr), _p64(oc), _pf(ov))
    if nnz < 0:
        raise MemoryError("oracle coo_to_csr allocation failed")
    return indptr, oc[:nnz].copy(), ov[:nnz].copy()


def weight_matrix(labels, k: int):
    """build_weight_matrix (embedding.py:92-107): the N x K one-hot CSR, row j
    holding 1.0 / n_{Y_j} at column Y_j, unlabeled rows empty."""
    lab = _i64(labels)
    counts = class_counts(lab, k)
    labeled = lab >= 0
    indptr = np.zeros(lab.size + 1, np.int64)
    np.cumsum(labeled, out=indptr[1:])
    cols = lab[labeled]
    return indptr, cols.astype(np.int64), 1.0 / counts[cols]


def to_csr(rows, cols, w, n: int, directed: bool):
    """EdgeList(n, rows, cols, w, directed).to_csr() (graph_io.py:78-92)."""
    r, c, v = symmetrize(rows, cols, w, directed)
    return coo_to_csr(r, c, v, n, n)


def add_identity(indptr, cols, data, n: int):
    """_kernels.py:169-198."""
    indptr, cols, data = _i64(indptr), _i64(cols), _f64(data)
    cap = data.size + n + 1
    oi = np.zeros(n + 1, np.int64)
    oc = np.empty(cap, np.int64)
    ov = np.empty(cap, np.float64)
    k = lib().gor_add_identity(_p64(indptr), _p64(cols), _pf(data), n, _p64(oi), _p64(oc), _pf(ov))
    return oi, oc[:k].copy(), ov[:k].copy()


def degree(indptr, data, n: int):
    """sparse.py:193-196 (bincount in storage order)."""
    indptr, data = _i64(indptr), _f64(data)
    d = np.empty(n, np.float64)
    lib().gor_degree(_p64(indptr), _pf(data), n, _pf(d))
    return d


def laplacian_normalize(indptr, cols, data, n: int, deg):
    """sparse.py:199-226; returns None on a negative degree."""
    indptr, cols, data, deg = _i64(indptr), _i64(cols), _f64(data), _f64(deg)
    oi = np.zeros(n + 1, np.int64)
    oc = np.empty(max(data.size, 1), np.int64)
    ov = np.empty(max(data.size, 1), np.float64)
    nnz = ctypes.c_int64(0)
    st = lib().gor_laplacian_normalize(_p64(indptr), _p64(cols), _pf(data), n, _pf(deg),
                                       _p64(oi), _p64(oc), _pf(ov), ctypes.byref(nnz))
    if st != OK:
        return None
    return oi, oc[: nnz.value].copy(), ov[: nnz.value].copy()


def class_counts(labels, k: int):
    """embedding.py:68-71."""
    labels = _i64(labels)
    out = np.zeros(k, np.int64)
    lib().gor_class_counts(_p64(labels), labels.size, k, _p64(out))
    return out


def spmm_onehot_dense(indptr, cols, data, labels, k: int):
    """spmm(A, build_weight_matrix(labels)).to_dense() (_kernels.py:257-307)."""
    indptr, cols, data, labels = _i64(indptr), _i64(cols), _f64(data), _i64(labels)
    n = labels.size
    counts = class_counts(labels, k)
    z = np.empty((n, k), np.float64)
    lib().gor_spmm_onehot_dense(_p64(indptr), _p64(cols), _pf(data), n, _p64(labels),
                                _p64(counts), k, _pf(z))
    return z


def correlate_rows(z):
    """embedding.py:134-143; returns None when z holds a non-finite value."""
    out = np.array(z, dtype=np.float64, copy=True, order="C")
    n, k = out.shape
    st = lib().gor_correlate_rows(_pf(out), n, k)
    return None if st != OK else out


def flags_of(laplacian: bool, diagonal: bool, correlation: bool) -> int:
    return (LAPLACIAN if laplacian else 0) | (DIAGONAL if diagonal else 0) | (
        CORRELATION if correlation else 0)


def encode_edges(rows, cols, w, n: int, directed: bool, labels, k: int, flags: int,
                 want_csr: bool = False, want_degree: bool = False):
    """encode(EdgeList(...).to_csr(), LabelVector, EmbedOptions) -- the whole
    reference timed region (cli.py:170-180).  Returns (status, z, extras)."""
    rows, cols, w, labels = _i64(rows), _i64(cols), _f64(w), _i64(labels)
    e = rows.size
    cap = max(e if directed else 2 * e, 1)
    z = np.empty((n, k), np.float64)
    extras = {}
    ip = oc = ov = dg = None
    nnz = ctypes.c_int64(0)
    if want_csr:
        ip = np.zeros(n + 1, np.int64)
        oc = np.empty(cap, np.int64)
        ov = np.empty(cap, np.float64)
    if want_degree:
        dg = np.zeros(n, np.float64)
    st = lib().gor_encode_edges(
        _p64(rows), _p64(cols), _pf(w), e, n, int(directed), _p64(labels), k, flags, _pf(z),
        _p64(ip) if ip is not None else None, _p64(oc) if oc is not None else None,
        _pf(ov) if ov is not None else None, ctypes.byref(nnz),
        _pf(dg) if dg is not None else None)
    if want_csr:
        extras["csr"] = (ip, oc[: nnz.value].copy(), ov[: nnz.value].copy())
    if want_degree:
        extras["degree"] = dg
    return st, z, extras
