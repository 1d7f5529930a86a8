"""Per-rank compute time of the row-sharded bitmap path on ONE GPU.

For P = 1, 2, 4, 8 the configs[1] graph is split into P equal-entry row
ranges (dist.shard_plan); the per-rank kernels of every shard (phase 1, then
phase 2 with the degree vector gathered by hand beforehand) are captured in
a CUDA graph and timed alone -- no collective, no other rank.  The maximum
over shards is the compute part of a P-GPU step; the NCCL all-gather of
the N uint32 degrees comes on top (not measurable with one GPU)."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_03726_b200 import _lib, dist as gdist, synth  # noqa: E402


def main():
    dev = torch.device("cuda")
    cfg = synth.make_config(1, device="cpu")
    n, k, flags = cfg["n"], cfg["k"], cfg["flags"]
    rows = torch.as_tensor(cfg["rows"], device=dev)
    cols = torch.as_tensor(cfg["cols"], device=dev)
    lab = torch.as_tensor(cfg["labels"], device=dev)
    out = {}
    for P in (1, 2, 4, 8):
        ranges = gdist.shard_plan(rows, cols, n, False, P)
        streams = [gdist.local_stream(rows, cols, None, False, rb, re) for rb, re in ranges]
        ops = [gdist.GpuShardOps(dev) for _ in ranges]
        deg_all = torch.cat([o.bm_degrees(s[0], s[1], n, rb, re, lab, k, flags)
                             for o, s, (rb, re) in zip(ops, streams, ranges)])
        times = []
        for o, s, (rb, re) in zip(ops, streams, ranges):
            def step():
                o.bm_degrees(s[0], s[1], n, rb, re, lab, k, flags)
                o.bm_encode(s[0], s[1], n, rb, re, k, flags, deg_all, check=False)
            for _ in range(3):
                step()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step()
            flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
            ts = []
            for _ in range(20):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                g.replay()
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b) * 1e3)
            ts.sort()
            # per-kernel breakdown (event records between launches, no PDL overlap)
            lib = _lib.load()
            ms_buf = (ctypes.c_float * 64)()
            nm_buf = (ctypes.c_char_p * 64)()
            brk = {}
            for _ in range(5):
                flush.zero_()
                lib.gee_profile_start(torch.cuda.current_stream().cuda_stream)
                step()
                lib.gee_profile_stop()
                got = lib.gee_profile_read(ms_buf, nm_buf, 64)
                for j in range(got):
                    brk.setdefault(nm_buf[j].decode(), []).append(ms_buf[j] * 1e3)
            brk = {kname: round(sorted(v)[len(v) // 2], 1) for kname, v in brk.items()}
            times.append({"rows": [rb, re], "entries": int(s[0].numel()), "us_median": ts[len(ts) // 2],
                          "kernels_us": brk})
        out[P] = {"shards": times, "max_us": max(t["us_median"] for t in times)}
        print(P, json.dumps(out[P]), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
