"""Seeded synthetic inputs for the five BASELINE.json configurations.

The paper's benchmark graphs (Network Repository) are not available, and the
reference ships only its SBM generator (sbm.py:115-155, a sequential numpy
PCG64 stream).  These generators stand in for them with the shapes, sizes and
value distributions BASELINE.json names ("Workloads").

Every random word is COUNTER-BASED -- word t of stream s is SplitMix64's
output for key mix64(seed ^ s * golden) -- so edge arrays are drawn on the
device by libgee's generator kernels (csrc/k_gen.cu) and the
reference arm draws the identical arrays on the host with the C restatement
(oracle/gee_gen.c).  Node-sized tables (labels, the Chung-Lu CDF) are built
here with numpy, for both arms.

  0  SBM       N=10,000  K=3   p_in=0.13 p_out=0.10, undirected, w=1.0   no options
  1  SBM       same graph                                                 lap+diag+corr
  2  Chung-Lu  N=600,000 E=1e7 exponent 2.5, w~U(0,1] f64, K=20 Zipf 1.1  lap+diag+corr
  3  R-MAT     N=2^24 E=2^28 (.57,.19,.19,.05) directed, dups kept,
               w~U(0,1] f32, K=50 uniform                                 lap+diag+corr
  4  G(n,m)    N=1e6 E=5e7 distinct pairs, w=1.0, K=1000 Zipf 1.5         lap+corr
"""

from __future__ import annotations

import numpy as np

LAP, DIAG, CORR = 1, 2, 4

CONFIGS = {
    0: dict(name="sbm_n10000_k3_plain", kind="sbm", n=10_000, k=3, p_in=0.13, p_out=0.10, seed=7,
            flags=0, directed=False),
    1: dict(name="sbm_n10000_k3_lap_diag_corr", kind="sbm", n=10_000, k=3, p_in=0.13, p_out=0.10,
            seed=7, flags=LAP | DIAG | CORR, directed=False),
    2: dict(name="chunglu_n600000_e1e7_k20", kind="chunglu", n=600_000, e=10_000_000, gamma=2.5,
            k=20, zipf=1.1, seed=2, flags=LAP | DIAG | CORR, directed=False),
    3: dict(name="rmat_s24_e2p28_k50_directed", kind="rmat", scale=24, e=1 << 28,
            abcd=(0.57, 0.19, 0.19, 0.05), k=50, seed=3, flags=LAP | DIAG | CORR, directed=True),
    4: dict(name="gnm_n1e6_e5e7_k1000", kind="gnm", n=1_000_000, e=50_000_000, k=1000, zipf=1.5,
            seed=4, flags=LAP | CORR, directed=False),
}

# stream ids of the counter-based generator
S_ROW, S_COL, S_W, S_LABEL, S_PERM, S_RMAT, S_PAIRS, S_SBM = 1, 2, 3, 4, 5, 6, 7, 8
_M64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15


def _mix64(z: int) -> int:
    z &= _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def stream_key(seed: int, stream: int) -> int:
    """mix64(seed ^ stream * golden): the key of one generator stream."""
    return _mix64(seed ^ ((stream * _GOLDEN) & _M64))


def draw_np(key: int, t: np.ndarray) -> np.ndarray:
    """Words t of stream `key` (uint64), vectorised: mix64(key + (t+1)*golden)."""
    with np.errstate(over="ignore"):
        z = np.uint64(key) + (t.astype(np.uint64) + np.uint64(1)) * np.uint64(_GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform_labels(seed: int, n: int, k: int) -> np.ndarray:
    """labels_i = hi32(word_i >> 32 * k): i.i.d. uniform over {0..k-1}."""
    hi = draw_np(stream_key(seed, S_LABEL), np.arange(n, dtype=np.uint64)) >> np.uint64(32)
    return ((hi * np.uint64(k)) >> np.uint64(32)).astype(np.int64)


def zipf_counts(n: int, k: int, s: float) -> np.ndarray:
    """Class sizes proportional to c^-s (c = 1..k), largest-remainder rounding
    (the apportionment of sbm.py:104-112)."""
    p = np.arange(1, k + 1, dtype=np.float64) ** (-s)
    p /= p.sum()
    raw = p * n
    base = np.floor(raw).astype(np.int64)
    short = n - int(base.sum())
    if short > 0:
        order = np.argsort(-(raw - base), kind="stable")
        base[order[:short]] += 1
    return base


def permuted_labels(seed: int, counts: np.ndarray) -> np.ndarray:
    """Labels with exactly `counts` members per class, placed by a random
    permutation (stable argsort of one word per node)."""
    n = int(counts.sum())
    lab = np.repeat(np.arange(counts.size, dtype=np.int64), counts)
    order = np.argsort(draw_np(stream_key(seed, S_PERM), np.arange(n, dtype=np.uint64)), kind="stable")
    out = np.empty(n, np.int64)
    out[order] = lab
    return out


def chunglu_cdf(n: int, gamma: float) -> np.ndarray:
    """CDF of p_i ~ (i+1)^(-1/(gamma-1)) (numpy cumsum, identical for both arms)."""
    w = (np.arange(n, dtype=np.float64) + 1.0) ** (-1.0 / (gamma - 1.0))
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    return cdf


def thresholds(probs) -> tuple:
    """Cumulative probabilities as 32-bit integer thresholds floor(P * 2^32)."""
    out, acc = [], 0.0
    for p in probs:
        acc += p
        out.append(min(int(acc * 4294967296.0), 0xFFFFFFFF))
    return tuple(out)


def spec(idx: int, scale_down: int = 0) -> dict:
    """Host-side description of config `idx`: sizes, options, labels and the
    generator parameters.  `scale_down` shrinks configs 2-4 by 2**scale_down
    in nodes (R-MAT: edges by 4**scale_down) for tests."""
    cfg = dict(CONFIGS[idx])
    kind, seed = cfg["kind"], cfg["seed"]
    if kind == "sbm":
        n = cfg["n"]
        cfg.update(labels=uniform_labels(seed, n, cfg["k"]), e=None, wdtype="unit",
                   thr=(min(int(cfg["p_in"] * 4294967296.0), 0xFFFFFFFF),
                        min(int(cfg["p_out"] * 4294967296.0), 0xFFFFFFFF)),
                   key=stream_key(seed, S_SBM))
    elif kind == "chunglu":
        n, e = cfg["n"] >> scale_down, cfg["e"] >> scale_down
        cfg.update(e=e, cdf=chunglu_cdf(n, cfg["gamma"]), wdtype="f64",
                   labels=permuted_labels(seed, zipf_counts(n, cfg["k"], cfg["zipf"])),
                   keys=(stream_key(seed, S_ROW), stream_key(seed, S_COL), stream_key(seed, S_W)))
    elif kind == "rmat":
        sc = cfg["scale"] - scale_down
        n = 1 << sc
        e = cfg["e"] >> (2 * scale_down)
        cfg.update(scale=sc, e=e, wdtype="f32", thr=thresholds(cfg["abcd"][:3]),
                   labels=uniform_labels(seed, n, cfg["k"]),
                   keys=(stream_key(seed, S_RMAT), stream_key(seed, S_W)))
    elif kind == "gnm":
        n, e = cfg["n"] >> scale_down, cfg["e"] >> scale_down
        cfg.update(e=e, wdtype="unit", labels=permuted_labels(seed, zipf_counts(n, cfg["k"], cfg["zipf"])),
                   key=stream_key(seed, S_PAIRS), limit=e + e // 32 + 4096)
    else:
        raise ValueError(kind)
    cfg["n"] = n
    cfg["idx"] = idx
    return cfg


def _device_edges(s: dict, dev):
    """Edge arrays of spec `s` drawn on the device by libgee (k_gen.cu)."""
    import torch

    from . import _device, _lib
    lib = _lib.load()
    st = _device.stream_handle()
    kind, n = s["kind"], s["n"]
    with torch.cuda.device(dev):
        if kind == "rmat":
            e = s["e"]
            rows = torch.empty(e, dtype=torch.int64, device=dev)
            cols = torch.empty(e, dtype=torch.int64, device=dev)
            w = torch.empty(e, dtype=torch.float32, device=dev)
            t1, t2, t3 = s["thr"]
            _lib.check(lib.gee_gen_rmat(s["keys"][0], s["keys"][1], s["scale"], e, t1, t2, t3,
                                        _device.ptr(rows), _device.ptr(cols), _device.ptr(w), st))
        elif kind == "chunglu":
            e = s["e"]
            cdf = torch.as_tensor(s["cdf"], device=dev)
            rows = torch.empty(e, dtype=torch.int64, device=dev)
            cols = torch.empty(e, dtype=torch.int64, device=dev)
            w = torch.empty(e, dtype=torch.float64, device=dev)
            rk, ck, wk = s["keys"]
            _lib.check(lib.gee_gen_chunglu(rk, ck, wk, _device.ptr(cdf), n, e, _device.ptr(rows),
                                           _device.ptr(cols), _device.ptr(w), st))
        elif kind == "gnm":
            e, lim = s["e"], s["limit"]
            keys = torch.empty(lim, dtype=torch.int64, device=dev)
            _lib.check(lib.gee_gen_pairs(s["key"], 0, lim, n, _device.ptr(keys), st))
            # first occurrence of each pair in candidate order (stable sort by key)
            sk, perm = torch.sort(keys, stable=True)
            first = torch.ones_like(sk, dtype=torch.bool)
            first[1:] = sk[1:] != sk[:-1]
            first &= sk >= 0
            keep = torch.zeros_like(first)
            keep[perm] = first
            idx = torch.nonzero(keep).flatten()
            if idx.numel() < e:
                raise RuntimeError("G(n,m) generator: not enough distinct candidate pairs")
            kept = keys[idx[:e]]
            rows, cols = kept // n, kept % n
            del keys, sk, perm, first, keep, idx, kept
            w = torch.ones(e, dtype=torch.float64, device=dev)
        elif kind == "sbm":
            lab = torch.as_tensor(s["labels"], device=dev)
            cnt = torch.empty(n, dtype=torch.int64, device=dev)
            ti, to = s["thr"]
            _lib.check(lib.gee_gen_sbm_count(s["key"], n, _device.ptr(lab), ti, to, _device.ptr(cnt), st))
            off = torch.zeros(n, dtype=torch.int64, device=dev)
            off[1:] = torch.cumsum(cnt, 0)[:-1]
            e = int((off[-1] + cnt[-1]).item())
            rows = torch.empty(e, dtype=torch.int64, device=dev)
            cols = torch.empty(e, dtype=torch.int64, device=dev)
            _lib.check(lib.gee_gen_sbm_fill(s["key"], n, _device.ptr(lab), ti, to, _device.ptr(off),
                                            _device.ptr(rows), _device.ptr(cols), st))
            w = torch.ones(e, dtype=torch.float64, device=dev)
        else:
            raise ValueError(kind)
    return rows, cols, w


def make_config(idx: int, device="cuda", scale_down: int = 0) -> dict:
    """Inputs of config `idx` on a CUDA device: dict(rows, cols, weights,
    labels, n, e, k, directed, flags, name, ...).  rows/cols/labels int64,
    weights float64 (float32 for config 3).  The host arrays of the same
    graph come from oracle/gen.py (C restatement, bit-identical)."""
    import torch
    s = spec(idx, scale_down)
    dev = torch.device(device)
    if dev.type != "cuda":
        raise ValueError("make_config draws on a CUDA device; host arrays: oracle.gen.host_config")
    rows, cols, w = _device_edges(s, dev)
    s.update(rows=rows, cols=cols, weights=w, labels=torch.as_tensor(s["labels"], device=dev),
             e=int(rows.shape[0]))
    return s
