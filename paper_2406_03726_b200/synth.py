"""Seeded synthetic inputs for the five BASELINE.json configurations.

The paper's benchmark graphs (Network Repository) are not available; these
generators stand in for them with the shapes, sizes and value distributions
BASELINE.json names ("Workloads").  All randomness is seeded;
numpy generators run on the host, the two largest graphs are drawn with a
seeded torch generator on the device (then copied to the host only when the
CPU oracle needs them).

  0  SBM       N=10,000  K=3   p_in=0.13 p_out=0.10, undirected, w=1.0   no options
  1  SBM       same graph                                                 lap+diag+corr
  2  Chung-Lu  N=600,000 E=1e7 exponent 2.5, w~U(0,1] f64, K=20 Zipf 1.1  lap+diag+corr
  3  R-MAT     N=2^24 E=2^28 (.57,.19,.19,.05) directed, dups kept,
               w~U(0,1] f32, K=50 uniform                                 lap+diag+corr
  4  G(n,m)    N=1e6 E=5e7 distinct pairs, w=1.0, K=1000 Zipf 1.5         lap+corr
"""

from __future__ import annotations

import numpy as np
import torch

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


def zipf_counts(n: int, k: int, s: float) -> np.ndarray:
    """Class sizes proportional to c^-s (c = 1..k), largest-remainder rounding."""
    p = np.arange(1, k + 1, dtype=np.float64) ** (-s)
    p /= p.sum()
    raw = p * n
    base = np.floor(raw).astype(np.int64)
    short = n - int(base.sum())
    if short > 0:
        order = np.argsort(-(raw - base), kind="stable")
        base[order[:short]] += 1
    return base


def sbm(n: int, k: int, p_in: float, p_out: float, seed: int, block: int = 1024):
    """Undirected SBM: labels i.i.d. uniform; each pair i<j is an edge with
    p_in (same class) or p_out.  Edges come out in row-major (i, j) order."""
    rng = np.random.default_rng(seed)
    labels = rng.integers(0, k, n).astype(np.int64)
    rows, cols = [], []
    for i0 in range(0, n - 1, block):
        i1 = min(n - 1, i0 + block)
        j0 = i0 + 1
        u = rng.random((i1 - i0, n - j0))
        p = np.where(labels[i0:i1, None] == labels[None, j0:], p_in, p_out)
        hit = u < p
        hit &= np.arange(j0, n)[None, :] > np.arange(i0, i1)[:, None]
        r, c = np.nonzero(hit)
        rows.append(r.astype(np.int64) + i0)
        cols.append(c.astype(np.int64) + j0)
    rows = np.concatenate(rows) if rows else np.empty(0, np.int64)
    cols = np.concatenate(cols) if cols else np.empty(0, np.int64)
    return rows, cols, labels


def chung_lu(n: int, e: int, gamma: float, seed: int):
    """E endpoint pairs drawn i.i.d. from p_i ~ (i+1)^(-1/(gamma-1));
    self-loops and duplicates kept (the reference sums them)."""
    rng = np.random.default_rng(seed)
    w = (np.arange(n, dtype=np.float64) + 1.0) ** (-1.0 / (gamma - 1.0))
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    rows = np.minimum(np.searchsorted(cdf, rng.random(e), side="right"), n - 1).astype(np.int64)
    cols = np.minimum(np.searchsorted(cdf, rng.random(e), side="right"), n - 1).astype(np.int64)
    weights = 1.0 - rng.random(e)  # (0, 1]
    return rows, cols, weights, rng


def rmat(scale: int, e: int, abcd, seed: int, device="cpu", chunk: int = 1 << 26):
    """R-MAT edges (no noise), directed, duplicates kept; float32 weights in (0, 1]."""
    a, b, c, _ = abcd
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    rows = torch.empty(e, dtype=torch.int64, device=device)
    cols = torch.empty(e, dtype=torch.int64, device=device)
    for s0 in range(0, e, chunk):
        m = min(chunk, e - s0)
        r = torch.zeros(m, dtype=torch.int64, device=device)
        q = torch.zeros(m, dtype=torch.int64, device=device)
        for _ in range(scale):
            u = torch.rand(m, generator=g, device=device)
            rb = (u >= a + b).to(torch.int64)
            cb = (((u >= a) & (u < a + b)) | (u >= a + b + c)).to(torch.int64)
            r = r * 2 + rb
            q = q * 2 + cb
        rows[s0:s0 + m] = r
        cols[s0:s0 + m] = q
    w = 1.0 - torch.rand(e, generator=g, device=device, dtype=torch.float32)
    return rows, cols, w, g


def gnm(n: int, m: int, seed: int, device="cpu"):
    """m distinct unordered pairs {i, j}, i != j, uniformly at random."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    keys = torch.empty(0, dtype=torch.int64, device=device)
    need = m
    while need > 0:
        draw = int(need * 1.05) + 1024
        i = torch.randint(0, n, (draw,), generator=g, device=device)
        j = torch.randint(0, n, (draw,), generator=g, device=device)
        ok = i != j
        lo = torch.minimum(i, j)[ok]
        hi = torch.maximum(i, j)[ok]
        keys = torch.unique(torch.cat([keys, lo * n + hi]))
        need = m - keys.numel()
    perm = torch.randperm(keys.numel(), generator=g, device=device)[:m]
    keys = keys[perm]
    return keys // n, keys % n, g


def make_config(idx: int, device="cpu", scale_down: int = 0):
    """Inputs of config `idx`: dict(rows, cols, weights, labels, n, k, directed,
    flags, name).  rows/cols/labels int64, weights float64 (float32 for
    cfg 3).  `scale_down` shrinks configs 2-4 by 2**scale_down (tests)."""
    cfg = dict(CONFIGS[idx])
    kind = cfg["kind"]
    if kind == "sbm":
        rows, cols, labels = sbm(cfg["n"], cfg["k"], cfg["p_in"], cfg["p_out"], cfg["seed"])
        n = cfg["n"]
        weights = np.ones(rows.shape[0])
    elif kind == "chunglu":
        n = cfg["n"] >> scale_down
        e = cfg["e"] >> scale_down
        rows, cols, weights, rng = chung_lu(n, e, cfg["gamma"], cfg["seed"])
        labels = rng.permutation(np.repeat(np.arange(cfg["k"], dtype=np.int64),
                                           zipf_counts(n, cfg["k"], cfg["zipf"])))
    elif kind == "rmat":
        sc = cfg["scale"] - scale_down
        n = 1 << sc
        e = cfg["e"] >> (2 * scale_down if scale_down else 0)
        rows, cols, weights, g = rmat(sc, e, cfg["abcd"], cfg["seed"], device)
        labels = torch.randint(0, cfg["k"], (n,), generator=g, device=device, dtype=torch.int64)
    elif kind == "gnm":
        n = cfg["n"] >> scale_down
        e = cfg["e"] >> scale_down
        rows, cols, g = gnm(n, e, cfg["seed"], device)
        weights = torch.ones(e, dtype=torch.float64, device=device)
        counts = zipf_counts(n, cfg["k"], cfg["zipf"])
        lab = np.repeat(np.arange(cfg["k"], dtype=np.int64), counts)
        perm = torch.randperm(n, generator=g, device=device)
        labels = torch.as_tensor(lab, device=device)[perm]
    else:
        raise ValueError(kind)
    cfg.update(rows=rows, cols=cols, weights=weights, labels=labels, n=n,
               e=int(rows.shape[0]))
    return cfg
