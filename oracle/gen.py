"""Host-side inputs of the BASELINE.json configurations -- TEST INFRASTRUCTURE ONLY.

Edge arrays come from oracle/gee_gen.c, the C restatement of libgee's
counter-based generator kernels (csrc/k_gen.cu), so the reference arm
(bench.py --impl reference), the CPU baseline and the full-size parity tests
see exactly the graph the device generators draw.  Node-sized tables
(labels, Chung-Lu CDF, thresholds, stream keys) come from
paper_2406_03726_b200.synth.spec, the single description both arms share.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import oracle as _O

_u64 = ctypes.c_uint64
_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_bound = False


def _lib():
    global _bound
    L = _O.lib()
    if not _bound:
        L.ggen_key.restype = _u64
        L.ggen_key.argtypes = [_u64, _u64]
        L.ggen_rmat.restype = None
        L.ggen_rmat.argtypes = [_u64, _u64, ctypes.c_int, _i64, ctypes.c_uint32, ctypes.c_uint32,
                                ctypes.c_uint32, _vp, _vp, _vp]
        L.ggen_chunglu.restype = None
        L.ggen_chunglu.argtypes = [_u64, _u64, _u64, _vp, _i64, _i64, _vp, _vp, _vp]
        L.ggen_pairs.restype = None
        L.ggen_pairs.argtypes = [_u64, _i64, _i64, _i64, _vp]
        L.ggen_gnm.restype = _i64
        L.ggen_gnm.argtypes = [_u64, _i64, _i64, _i64, _vp, _vp]
        L.ggen_sbm.restype = _i64
        L.ggen_sbm.argtypes = [_u64, _i64, _vp, ctypes.c_uint32, ctypes.c_uint32, _vp, _vp]
        _bound = True
    return L


def _p(a):
    return a.ctypes.data_as(_vp) if a is not None else None


def host_edges(s: dict):
    """(rows int64, cols int64, weights) of spec `s` (synth.spec) on the host;
    weights float32 for R-MAT, float64 otherwise (ones for unit-weight graphs)."""
    L = _lib()
    kind, n = s["kind"], s["n"]
    if kind == "rmat":
        e = s["e"]
        rows, cols = np.empty(e, np.int64), np.empty(e, np.int64)
        w = np.empty(e, np.float32)
        t1, t2, t3 = s["thr"]
        L.ggen_rmat(s["keys"][0], s["keys"][1], s["scale"], e, t1, t2, t3, _p(rows), _p(cols), _p(w))
    elif kind == "chunglu":
        e = s["e"]
        rows, cols = np.empty(e, np.int64), np.empty(e, np.int64)
        w = np.empty(e, np.float64)
        cdf = np.ascontiguousarray(s["cdf"], np.float64)
        rk, ck, wk = s["keys"]
        L.ggen_chunglu(rk, ck, wk, _p(cdf), n, e, _p(rows), _p(cols), _p(w))
    elif kind == "gnm":
        e = s["e"]
        rows, cols = np.empty(e, np.int64), np.empty(e, np.int64)
        if L.ggen_gnm(s["key"], n, e, s["limit"], _p(rows), _p(cols)) < 0:
            raise RuntimeError("G(n,m) generator: not enough distinct candidate pairs")
        w = np.ones(e, np.float64)
    elif kind == "sbm":
        lab = np.ascontiguousarray(s["labels"], np.int64)
        ti, to = s["thr"]
        e = L.ggen_sbm(s["key"], n, _p(lab), ti, to, None, None)
        rows, cols = np.empty(e, np.int64), np.empty(e, np.int64)
        L.ggen_sbm(s["key"], n, _p(lab), ti, to, _p(rows), _p(cols))
        w = np.ones(e, np.float64)
    else:
        raise ValueError(kind)
    return rows, cols, w


def host_config(idx: int, scale_down: int = 0) -> dict:
    """synth.spec(idx) plus its host edge arrays (rows, cols, weights, labels)."""
    from paper_2406_03726_b200 import synth
    s = synth.spec(idx, scale_down)
    rows, cols, w = host_edges(s)
    s.update(rows=rows, cols=cols, weights=w, e=int(rows.shape[0]))
    return s


def pairs(key: int, t0: int, count: int, n: int) -> np.ndarray:
    """Raw G(n,m) candidate keys (for the generator kernel's parity test)."""
    out = np.empty(count, np.int64)
    _lib().ggen_pairs(key, t0, count, n, _p(out))
    return out
