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
