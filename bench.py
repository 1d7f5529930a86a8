#!/usr/bin/env python3
"""Benchmark: GEE edges/sec on B200 (BASELINE.json metric), one JSON line.

Step = one pass of the reference's timed region (cli.py:170-180:
``encode(edges.to_csr(), labels, opts)``) over the configuration's edge
list: device edge list + labels -> Z (N x K float64), i.e. label histogram,
CSR assembly (+ fused degrees), fused embedding.  Inputs are resident in HBM
when the timed region starts; L2 is flushed (512 MiB write) before every
timed step.  `value` = input edges / device time per step (CUDA events on
the launching stream, max over ranks); `e2e` = the same metric through
GeeEncoder.run_host (pinned host in -> pinned host Z out, copies timed).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C]
  python bench.py --impl reference ...   # the CPU reference (oracle port)

Under torchrun (N > 1) the rows are sharded across ranks
(paper_2406_03726_b200/dist.py); only rank 0 prints.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GEE edges/sec"
UNIT = "edges/s"
# sparse GEE, SBM 10k nodes / ~5.6M edges / K=3, Lap+Diag+Corr: 0.6 s
# on a 2 GHz quad-core i5 laptop -> the only published
# number for a benchmark configuration (configs[1]).
PUBLISHED = {1: 5.6e6 / 0.6}
FALLBACK_HBM_GBS = 6650.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", type=int, default=3,
                   help="BASELINE.json configs[C]; default 3, the metric's multi-GPU R-MAT workload "
                        "(the largest that fits one GPU)")
    p.add_argument("--impl", choices=["b200", "reference"], default="b200")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--fp32", action="store_true", help="the optional fp32 path: Z stored as float32 (1e-5)")
    p.add_argument("--permute-edges", action="store_true", help="side measurement: seeded random edge order")
    p.add_argument("--weighted", action="store_true", help="side measurement: U(0,1] f64 weights instead of 1.0")
    p.add_argument("--stream-variant", type=int, default=0,
                   help="debug A/B of the stream embed (results wrong by design): 1 no shared atomics, 2 no gathers")
    p.add_argument("--stream-tile-kb", type=int, default=0, help="debug: KB of the stream encode's Z tile")
    p.add_argument("--stream-nt", type=int, default=None,
                   help="retired debug knob (the stream embed is built for 128-thread CTAs only)")
    p.add_argument("--no-stream", action="store_true",
                   help="debug: disable the bucketed stream encode (gee_debug_set GEE_DEBUG_STREAM=1): exact CSR path")
    p.add_argument("--eager", action="store_true", help="launch kernels one by one instead of a CUDA graph")
    p.add_argument("--flush-mib", type=int, default=512)
    p.add_argument("--flush-mode", choices=("write", "clean"), default="write",
                   help="L2 flush between timed steps: write the buffer (default), or write it and then read "
                        "a second one so the flush's dirty lines are written back before the step")
    p.add_argument("--cpu-budget-s", type=float, default=12.0)
    p.add_argument("--cpu-sample-edges", type=int, default=1 << 25,
                   help="cpu_baseline: time the oracle on the first S edges of the workload when it has more")
    p.add_argument("--ref-budget-s", type=float, default=300.0,
                   help="--impl reference: stop after this many seconds of timed runs (at least one run)")
    p.add_argument("--embed-flat-bytes", type=int, default=None,
                   help="debug: per-warp shared budget of the K > 8 embed's flat row blocks "
                        "(gee_debug_set GEE_DEBUG_EMBED_FLAT_BYTES; 0 = one warp per row)")
    p.add_argument("--embed-flat-rowmax", type=int, default=None,
                   help="debug: longest row a flat embed block takes (GEE_DEBUG_EMBED_FLAT_ROWMAX)")
    p.add_argument("--force-path", type=int, default=0,
                   help="debug: CSR assembly path hook (gee_debug_set GEE_DEBUG_FORCE_BUCKETS)")
    p.add_argument("--shuffle", action="store_true",
                   help="sharded step from per-rank slices of the edge list: device row histogram, "
                        "all-reduce, partition and all-to-all edge shuffle inside the timed region "
                        "(dist.encode_distributed; implies --sharded)")
    p.add_argument("--sharded", action="store_true",
                   help="run the row-sharded multi-GPU step even with one rank (exercises dist.py under NCCL)")
    return p.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def workload_desc(c):
    opts = [n for b, n in ((1, "laplacian"), (2, "diagonal"), (4, "correlation")) if c["flags"] & b]
    return {
        "workload": f"configs[{c['idx']}] {c['name']}",
        "n_nodes": int(c["n"]), "n_edges": int(c["e"]), "k_classes": int(c["k"]),
        "directed": bool(c["directed"]), "options": opts or ["none"],
        "weights": "unit (1.0)" if c.get("wdtype") == "unit" else str(c.get("wdtype")),
        "seed": c["seed"],
        "step": "edge list + labels -> Z (EdgeList.to_csr + encode, cli.py:170-180)",
    }


def load_config(idx, device):
    """Config `idx`: drawn on the GPU by libgee's counter-based generators, or
    (device "cpu") on the host by their C restatement (oracle/gee_gen.c) --
    the same arrays bit for bit (tests/test_gpu_gen.py), so both arms time the
    same graph."""
    import torch
    if str(device) == "cpu":
        from oracle import gen
        return gen.host_config(idx)
    from paper_2406_03726_b200 import synth
    return synth.make_config(idx, device=torch.device(device))


def apply_variant(c, args):
    """Workload variants for the side measurements (never the default line):
    --permute-edges: the same edge list in a seeded random order (the SBM
    generator emits row-major order); --weighted: U(0,1] float64 weights
    instead of 1.0 (the general weighted paths instead of the unit-weight ones)."""
    import torch
    if not (args.permute_edges or args.weighted):
        return c
    c = dict(c)
    e = int(c["e"])
    if args.permute_edges:
        g = torch.Generator(device=c["rows"].device).manual_seed(12345)
        perm = torch.randperm(e, generator=g, device=c["rows"].device)
        c["rows"], c["cols"] = c["rows"][perm], c["cols"][perm]
        if c["weights"] is not None:
            c["weights"] = c["weights"][perm]
    if args.weighted:
        g = torch.Generator(device=c["rows"].device).manual_seed(54321)
        c["weights"] = 1.0 - torch.rand(e, generator=g, device=c["rows"].device, dtype=torch.float64)
        c["wdtype"] = "f64"
    c["variant"] = ",".join(v for v, on in (("permuted edge order", args.permute_edges),
                                            ("U(0,1] f64 weights", args.weighted)) if on)
    return c


def host_arrays(c):
    import torch
    out = []
    for key in ("rows", "cols", "weights", "labels"):
        x = c[key]
        out.append(x.cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x))
    return out


# ---------------------------------------------------------------------------
# CPU reference arm (oracle port of the reference pipeline)
# ---------------------------------------------------------------------------
def cpu_reference_time(arrays, c, budget_s, min_reps=1, max_reps=5, sample=None):
    """Seconds per run of the C restatement of the reference pipeline
    (encode(EdgeList(...).to_csr(), ...), cli.py:170-180) on these host
    arrays; `sample` = time only the first S edges (same N, K, options)."""
    from oracle import oracle as O
    rows, cols, w, labels = arrays
    if sample is not None and sample < rows.shape[0]:
        rows, cols, w = rows[:sample], cols[:sample], w[:sample]
    w = np.asarray(w, dtype=np.float64)  # EdgeList promotes float32 (graph_io.py:61)
    times = []
    t_start = time.perf_counter()
    while len(times) < max_reps:
        t0 = time.perf_counter()
        st, _, _ = O.encode_edges(rows, cols, w, c["n"], c["directed"], labels, c["k"], c["flags"])
        times.append(time.perf_counter() - t0)
        if st != O.OK:
            raise RuntimeError(f"oracle status {st}")
        if len(times) >= min_reps and time.perf_counter() - t_start > budget_s:
            break
    return times, int(rows.shape[0])


def run_reference(args):
    """The reference arm: the CPU reference pipeline (its C restatement,
    oracle/gee_oracle.c, pinned bitwise to the reference) on the FULL
    workload of --config, drawn on the host by oracle/gee_gen.c.  The C code
    has no JIT, so warm-up runs are not needed and none are made; timed runs
    stop at --steps or once --ref-budget-s has elapsed (at least one), and
    `steps` reports the runs actually made."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    c = load_config(args.config, "cpu")
    arrays = host_arrays(c)
    times, e = cpu_reference_time(arrays, c, args.ref_budget_s, 1, max(1, args.steps))
    t = statistics.mean(times)
    value = e / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": len(times), "steps_requested": args.steps, "warmup": 0,
        "warmup_requested": args.warmup,
        "ms_per_step": t * 1e3, "ms_per_step_min": min(times) * 1e3, "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": (value / PUBLISHED[args.config]) if args.config in PUBLISHED else None,
        "dtype": "f64" + ("; Z stored f32 (--fp32)" if args.fp32 else ""),
        "data": "synthetic (seeded counter-based generator, BASELINE.json shapes)",
        "config": workload_desc(c),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": f"full configs[{args.config}] workload ({e} edges), {len(times)} timed "
                                   "runs of the C restatement of the reference pipeline "
                                   "(oracle/gee_oracle.c; the reference is single-threaded, numba @njit "
                                   "without parallel, so 1 core)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML, sampled every 5 ms)
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting",
        0x1: "gpu_idle",
    }

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], set(), False
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
        self._stop = threading.Event()

    def _loop(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": len(self.samples)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# algorithmic bytes per launch
# ---------------------------------------------------------------------------
def kernel_bytes(c, m_stream, nnz, wbytes, zbytes=8):
    """Compulsory bytes each kernel must move once.
    wbytes = bytes per weight actually read (0 for unit-weight graphs, whose
    values are implicit 1.0 and never stored or read)."""
    n, e, k = int(c["n"]), int(c["e"]), int(c["k"])
    lap = bool(c["flags"] & 1)
    directed = bool(c["directed"])
    rb = (max(n - 1, 1)).bit_length() if directed else n.bit_length()
    keybits = rb + (max(n - 1, 1)).bit_length()
    kb = 8 if keybits > (31 if directed else 32) else 4  # sort key bytes
    vb = 8 if wbytes else 0  # stored CSR value bytes per entry
    np_ = (n + 255) // 256 * 256
    bm = np_ * np_ // 8
    nbx = 16 if 7 * k <= 16 else 32 if 7 * k <= 32 else 64  # X digit columns (k_bitmap.cu)
    return {
        # bitmap path (unit weights, N <= 16384): the edge list is the only
        # HBM stream; the Np x Np adjacency bitmap (Np = n rounded up to 256)
        # lives in L2 and is counted once per pass over it
        "k_bm_set": 16 * e + 8 * n,
        "k_bm_sym": 2 * bm + 4 * n,
        "k_bm_table": 4 * n + 4 * n + 9 * n + 7 * n + (16 * n if lap else 0),
        "k_bm_scan": bm + 4 * n + 9 * n + (16 * n if lap else 0),
        "k_bm_gemm": bm + nbx * np_ + 8 * n * k + 4 * n + (8 * n if lap else 0),
        # radix-sort path (k_sort.cu): key width as sort_keybits / sort_wide_key,
        # payload = the weight in its own width (none for unit weights)
        "k_sort_hist": (16 + wbytes) * e,
        "k_onesweep": 2 * m_stream * (kb + wbytes),
        "k_dedup": m_stream * (kb + wbytes) + (4 + vb) * nnz + 16 * (n + 1),
        "k_degree": (4 + vb) * nnz + 8 * (n + 1) + (16 * n if lap else 8 * n),
        # bucket path
        "k_count_part": 16 * e,
        "k_count_global": 16 * e,
        "k_scatter_part": (16 + wbytes) * e + 16 * m_stream,
        "k_scatter_global": (16 + wbytes) * e + 16 * m_stream + 8 * n,
        "k_rows": 16 * m_stream + 8 * (n + 1) + (4 + vb) * nnz + 4 * n + (16 * n if lap else 0),
        # embed: col (+val) per stored entry, row extents, one 16-B node record
        # per node, the row scale, and Z
        "k_embed": (4 + vb) * nnz + 8 * (n + 1) + 4 * n + 16 * n + (8 * n if lap else 0) + 8 * n * k,
        "k_label_hist": 8 * n + 4 * n,
        # bucketed stream encode (k_stream.cu): M = stream entries, wbytes the
        # weight width (0 unit); keys1 8 B, keys2 4 B per entry
        "k_st_hist1": (8 if directed else 16) * e,
        "k_st_part1": (16 + wbytes) * e + (8 + wbytes) * m_stream,
        "k_st_hist2": 8 * m_stream,
        "k_st_part2": (8 + wbytes) * m_stream + (4 + wbytes) * m_stream,
        "k_st_degree": ((4 + wbytes) * m_stream + 8 * n if lap else 0) + 4 * n + 8 * n + 16 * n,
        # the fused SpMM + normalisation kernel: entries once, one node record
        # per node, the row scales, Z written once
        "k_st_embed": (4 + wbytes) * m_stream + 16 * n + (8 * n if lap else 0) + zbytes * n * k,
        "k_node_rec": 4 * n + 16 * n + (8 * n if lap else 0),
    }


def _traffic(cfg, kernel):
    """ncu dram__bytes_read.sum + dram__bytes_write.sum per launch for this
    kernel at this config (profiles/traffic.json, from an ncu --set full
    capture), or None."""
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(tpath)).get(f"cfg{cfg}", {}).get(kernel)
    except Exception:
        return None


def _kernel_table(lib, per_kernel, steps, models, prof_total):
    import statistics as st_
    ktab = []
    for name, ts in per_kernel.items():
        t_launch = st_.mean(ts)
        bts = models.get(name)
        ktab.append({"kernel": name, "ms_per_launch": t_launch, "launches_per_step": len(ts) / steps,
                     "share": sum(ts) / prof_total, "alg_bytes": bts,
                     "gbs": (bts / (t_launch * 1e-3) / 1e9) if bts else None})
    ktab.sort(key=lambda r: -r["share"])
    return ktab


def _profile_steps(lib, fn, steps):
    """Per-kernel device times of `steps` eager runs of fn (event marks between launches)."""
    import ctypes
    import torch
    cap = 256
    ms_buf = (ctypes.c_float * cap)()
    nm_buf = (ctypes.c_char_p * cap)()
    per_kernel, totals = {}, []
    for _ in range(steps):
        lib.gee_profile_start(torch.cuda.current_stream().cuda_stream)
        fn()
        lib.gee_profile_stop()
        got = lib.gee_profile_read(ms_buf, nm_buf, cap)
        if got < 0:
            raise RuntimeError("gee_profile_read: " + lib.gee_last_error_string().decode())
        totals.append(sum(ms_buf[j] for j in range(got)))
        for j in range(got):
            per_kernel.setdefault(nm_buf[j].decode(), []).append(ms_buf[j])
    return per_kernel, sum(totals)


def run_sharded(args, rank, world, local, dev):
    """The row-sharded step on `world` GPUs (one process each, NCCL): every
    rank draws the same seeded graph and keeps the stream entries of its row
    range (equal entries per rank; outside the timed region).  Step =
    partition + degrees of the rank's rows, ALL-GATHER of the degree vector
    (Laplacian), node table + fused embed of the rank's rows.  value = input
    edges / max over ranks of the mean step time (strong scaling: the whole
    graph is split)."""
    import torch
    import torch.distributed as dist

    from paper_2406_03726_b200 import _lib
    from paper_2406_03726_b200 import dist as gdist
    lib = _lib.load()
    c = load_config(args.config, dev)
    n, e, k, directed, flags = c["n"], c["e"], c["k"], c["directed"], c["flags"]
    rows, cols, lab = c["rows"], c["cols"], c["labels"]
    w = c["weights"]
    if c.get("wdtype") == "unit":
        w = None
    ranges = gdist.shard_plan(rows, cols, n, directed, world)
    rb, re = ranges[rank]
    stream = gdist.local_stream(rows, cols, w, directed, rb, re)
    e_local = int(stream[0].numel())
    ops = gdist.GpuShardOps(dev)
    nonneg = gdist.stream_ok(w)
    use_bm = ops.bitmap_ok(n, k, w is not None)
    mode = "bitmap" if use_bm else ("stream" if nonneg else "csr")
    z_out = torch.empty((re - rb, k), dtype=torch.float64, device=dev)
    if mode == "stream":
        def step():
            return gdist.encode_rows_stream(ops, stream, lab, n, k, flags, ranges, rank, check=False, z=z_out)
    elif mode == "bitmap":
        def step():
            return gdist.encode_rows_bitmap(ops, stream, lab, n, k, flags, ranges, rank, check=False)
    else:
        def step():
            return gdist.encode_rows(ops, stream, lab, n, k, flags, ranges, rank)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    run, graphed = step, False
    if mode != "csr" and not args.eager:
        try:  # the whole rank step, kernels and the NCCL all-gather, as one CUDA graph
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step()
            run, graphed = g.replay, True
            run()
            torch.cuda.synchronize()
        except Exception as ex:
            print(f"[rank {rank}] CUDA graph capture failed ({ex}); timing eager launches", file=sys.stderr)
            run, graphed = step, False
    lib.gee_reset_launch_count()
    step()
    torch.cuda.synchronize()
    launches_per_step = int(lib.gee_launch_count())
    sampler = ClockSampler(local) if rank == 0 else None
    times = []
    if sampler:
        sampler.__enter__()
    for _ in range(args.steps):
        dist.barrier()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        run()
        s1.record()
        torch.cuda.synchronize()
        times.append(s0.elapsed_time(s1))
    if sampler:
        sampler.__exit__()
    dist.barrier()
    if mode == "stream":
        ops.st_check()
    elif mode == "bitmap":
        _lib.raise_device_errors(int(ops._bm_err.item()), "sharded bitmap encode")
    ms_t = torch.tensor([statistics.mean(times)], device=dev)
    dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t)
    # per-kernel breakdown of this rank's step (eager, event marks between launches)
    per_kernel, prof_total = _profile_steps(lib, step, max(1, min(args.steps, 5)))
    m_local = e_local
    models = kernel_bytes(dict(c, n=n, e=e_local, directed=True), m_local, m_local,
                          0 if w is None else w.element_size())
    # the rank's embed covers only its rows: Z bytes of (re - rb) rows, node records of all n
    if "k_st_embed" in models:
        wb = 0 if w is None else w.element_size()
        lap = bool(flags & 1)
        models["k_st_embed"] = (4 + wb) * m_local + 16 * n + (8 * n if lap else 0) + 8 * (re - rb) * k
    ktab = _kernel_table(lib, per_kernel, max(1, min(args.steps, 5)), models, prof_total)
    hbm, peak_src = peaks()
    emb = next((r for r in ktab if r["kernel"] in ("k_st_embed", "k_embed")), None)
    dom = next((r for r in ktab if r["alg_bytes"]), None)
    # end to end: this rank's pinned host entries up, its step, its Z rows down
    e2e = None
    if not args.no_e2e:
        hs = [None if x is None else x.cpu().pin_memory() for x in stream]
        zh = torch.empty((re - rb, k), dtype=torch.float64).pin_memory()
        ds = list(stream)
        dist.barrier()
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(args.steps):
            for h, d in zip(hs, ds):
                if h is not None:
                    d.copy_(h, non_blocking=True)
            zz = step()
            zh.copy_(zz, non_blocking=True)
        t1.record()
        torch.cuda.synchronize()
        e2e_t = torch.tensor([t0.elapsed_time(t1) / args.steps], device=dev)
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
        h2d = sum(h.numel() * h.element_size() for h in hs if h is not None)
        e2e = {"value": e / (float(e2e_t) * 1e-3), "unit": UNIT, "ms_per_step": float(e2e_t),
               "h2d_bytes_per_step": int(h2d) * world, "d2h_bytes_per_step": int(zh.numel() * 8) * world,
               "api": "per rank: pinned host stream slice in, the rank step, its Z rows out (max over ranks)"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        arrays = host_arrays(c)
        tms, es = cpu_reference_time(arrays, c, args.cpu_budget_s, 1, 5, sample=args.cpu_sample_edges)
        cpu = {"value": es / statistics.mean(tms), "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"the first {es} of the {e} edges of configs[{args.config}], C restatement, 1 core"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": e / (ms * 1e-3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": (e / (ms * 1e-3) / PUBLISHED[args.config]) if args.config in PUBLISHED else None,
            "dtype": "f64", "data": "synthetic (seeded counter-based generator, BASELINE.json shapes)",
            "config": workload_desc(c),
            "workload_detail": {"parallelism": f"row-sharded x{world} ({mode} path): equal stream entries per "
                                               "rank; NCCL all-gather of the degree vector (Laplacian)",
                                "rank0_rows": [rb, re], "rank0_entries": e_local, "cuda_graph": graphed},
            "roofline": ({"bound": "hbm", "kernel": dom["kernel"], "achieved": dom["gbs"], "peak": hbm,
                          "peak_source": peak_src, "unit": "GB/s", "frac": dom["gbs"] / hbm,
                          "traffic": _traffic(args.config, dom["kernel"]), "alg_bytes_per_launch": dom["alg_bytes"],
                          "scope": "rank 0's kernels"} if dom else None),
            "embed_kernel": ({"kernel": emb["kernel"], "ms_per_launch": emb["ms_per_launch"], "gbs": emb["gbs"],
                              "frac": emb["gbs"] / hbm} if emb and emb["gbs"] else None),
            "kernels": ktab,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "launch_mode": "cuda_graph (kernels + NCCL, one replay per step)" if graphed else "eager",
            "clocks": sampler.summary() if sampler else None,
        }
        sys.stdout.flush()
        os.write(_REAL_STDOUT if _REAL_STDOUT is not None else 1, (json.dumps(line) + "\n").encode())
    dist.barrier()
    dist.destroy_process_group()
    return 0


_REAL_STDOUT = None


def run_b200(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or args.sharded or args.shuffle:
        # NCCL may print its banner on stdout: keep stdout for the JSON line only
        global _REAL_STDOUT
        sys.stdout.flush()
        _REAL_STDOUT = os.dup(1)
        os.dup2(2, 1)
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
        if args.shuffle:
            from paper_2406_03726_b200 import dist as gdist
            return gdist.bench_sharded(args, rank, world, dev)
        return run_sharded(args, rank, world, local, dev)

    import paper_2406_03726_b200 as G
    from paper_2406_03726_b200 import _lib

    lib = _lib.load()
    if args.force_path:
        lib.gee_debug_set(_lib.DEBUG_FORCE_BUCKETS, args.force_path)
    if args.no_stream:
        lib.gee_debug_set(_lib.DEBUG_STREAM, 1)
    if args.stream_tile_kb:
        lib.gee_debug_set(5, args.stream_tile_kb)
    if args.stream_nt is not None:
        lib.gee_debug_set(6, args.stream_nt)
    if args.stream_variant:
        lib.gee_debug_set(_lib.DEBUG_STREAM, 16 + args.stream_variant)
    if args.embed_flat_bytes is not None:
        lib.gee_debug_set(_lib.DEBUG_EMBED_FLAT_BYTES, args.embed_flat_bytes)
    if args.embed_flat_rowmax is not None:
        lib.gee_debug_set(_lib.DEBUG_EMBED_FLAT_ROWMAX, args.embed_flat_rowmax)
    c = apply_variant(load_config(args.config, dev), args)
    n, e, k, directed, flags = c["n"], c["e"], c["k"], c["directed"], c["flags"]
    rows = torch.as_tensor(c["rows"], device=dev)
    cols = torch.as_tensor(c["cols"], device=dev)
    w_in = torch.as_tensor(c["weights"], device=dev)
    lab = torch.as_tensor(c["labels"], device=dev)
    # the public container validates the edge list (outside the timed region,
    # as the reference's EdgeList does) and notes unit weights
    edges = G.EdgeList(n, rows, cols, w_in, directed)
    _, w = edges.weight_kind()  # None for unit-weight graphs: never re-read
    opts = G.EmbedOptions(bool(flags & 1), bool(flags & 2), bool(flags & 4))
    enc = G.GeeEncoder(n, e, k, directed, opts, dev, nonneg=bool(edges.nonneg),
                       dtype=torch.float32 if args.fp32 else torch.float64)
    flush_buf = torch.empty(args.flush_mib << 20, dtype=torch.uint8, device=dev)
    clean_buf = torch.zeros(args.flush_mib << 20 if args.flush_mode == "clean" else 0, dtype=torch.uint8,
                            device=dev)

    class _Flush:
        # "write": the flush buffer is written (L2 left full of its dirty lines,
        # whose write-back then lands inside the next step); "clean": written,
        # then a second buffer of the same size is read, so the write-back
        # happens here and the step starts from a cold, clean L2
        @staticmethod
        def zero_():
            flush_buf.zero_()
            if clean_buf.numel():
                clean_buf.max()

    flush = _Flush()
    # stream length and unique nnz for the byte model (outside the timed region)
    m_stream = e if directed else e + int((rows != cols).sum().item())
    nnz = edges.to_csr().nnz
    wbytes = 0 if w is None else w.element_size()

    enc.run(rows, cols, w, lab, check=True)  # surfaces any data error once
    lib.gee_reset_launch_count()
    enc.run(rows, cols, w, lab, check=False)
    launches_per_step = int(lib.gee_launch_count())
    if not args.eager:
        # the whole step as one CUDA graph (no host launch gaps); a second
        # capture carries an event-record node after every kernel for the
        # per-kernel breakdown
        g_plain = enc.capture(rows, cols, w, lab, profile=False)
        g_prof = enc.capture(rows, cols, w, lab, profile=True)
        step_fn, prof_fn = g_plain.replay, g_prof.replay
    else:
        def step_fn():
            enc.run(rows, cols, w, lab, check=False)

        def prof_fn():
            lib.gee_profile_start(torch.cuda.current_stream().cuda_stream)
            enc.run(rows, cols, w, lab, check=False)
            lib.gee_profile_stop()
    for _ in range(args.warmup):
        flush.zero_()
        step_fn()
        flush.zero_()
        prof_fn()
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    per_kernel = {}
    import ctypes
    cap = 256
    ms_buf = (ctypes.c_float * cap)()
    nm_buf = (ctypes.c_char_p * cap)()
    sampler = ClockSampler(local)
    torch.cuda.synchronize()
    with sampler:
        # timed region: K steps, L2 flushed before each, CUDA events around each
        for i in range(args.steps):
            flush.zero_()
            starts[i].record(stream)
            step_fn()
            ends[i].record(stream)
        torch.cuda.synchronize()
        # per-kernel breakdown: the same step with event records between kernels
        prof_steps = []
        for i in range(args.steps):
            flush.zero_()
            prof_fn()
            got = lib.gee_profile_read(ms_buf, nm_buf, cap)
            if got < 0:
                raise RuntimeError("gee_profile_read: " + lib.gee_last_error_string().decode())
            prof_steps.append(sum(ms_buf[j] for j in range(got)))
            for j in range(got):
                per_kernel.setdefault(nm_buf[j].decode(), []).append(ms_buf[j])
        torch.cuda.synchronize()
    launches = launches_per_step * args.steps
    step_ms = [s.elapsed_time(t) for s, t in zip(starts, ends)]
    _device_err = int(enc.err.item())
    ms = statistics.mean(step_ms)
    value = e / (ms * 1e-3)

    # roofline of the dominant kernel (largest share of the step)
    hbm, peak_src = peaks()
    models = kernel_bytes(c, m_stream, nnz, wbytes, 4 if args.fp32 else 8)
    ktab = []
    for name, ts in per_kernel.items():
        launches_per_step = len(ts) / args.steps
        t_launch = statistics.mean(ts)
        b = models.get(name)
        ktab.append({"kernel": name, "ms_per_launch": t_launch, "launches_per_step": launches_per_step,
                     "share": sum(ts) / sum(prof_steps),
                     "alg_bytes": b, "gbs": (b / (t_launch * 1e-3) / 1e9) if b else None})
    ktab.sort(key=lambda r: -r["share"])
    dom = next(r for r in ktab if r["alg_bytes"])
    traffic = _traffic(args.config, dom["kernel"])
    roofline = {"bound": "hbm", "kernel": dom["kernel"], "achieved": dom["gbs"], "peak": hbm,
                "peak_source": peak_src, "unit": "GB/s", "frac": dom["gbs"] / hbm,
                "traffic": traffic, "alg_bytes_per_launch": dom["alg_bytes"]}
    emb = next((r for r in ktab if r["kernel"] in ("k_st_embed", "k_embed")), None)
    prod = next((r for r in ktab if r["kernel"] in ("k_bm_gemm", "k_st_embed", "k_embed")), None)

    # end to end: pinned host in -> Z on host, through the public plan API
    e2e = None
    if not args.no_e2e:
        rh, ch, wh, lh = host_arrays(c)
        h2d, d2h = enc.attach_host(rh, ch, None if w is None else wh, lh, depth=2)
        enc.run_host(check=True)
        torch.cuda.synchronize()
        # (1) the synchronous call: copies in, pipeline, Z out, one step at a time
        es = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ee = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        for i in range(args.steps):
            es[i].record(stream)
            enc.run_host(check=False)
            ee[i].record(stream)
        torch.cuda.synchronize()
        serial_ms = statistics.mean(a.elapsed_time(b) for a, b in zip(es, ee))
        # (2) a stream of encodes through run_host_async: step i's Z download
        # overlaps step i+1's input upload (full-duplex PCIe); every step still
        # copies its inputs up and its Z down inside the timed region
        for _ in range(2):
            enc.run_host_async()
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        enc._s_in.wait_stream(stream)
        last = None
        for i in range(args.steps):
            _, last = enc.run_host_async()
        enc._s_out.wait_event(last)
        t1.record(enc._s_out)
        torch.cuda.synchronize()
        pipe_ms = t0.elapsed_time(t1) / args.steps
        _device_err2 = int(enc.err.item())
        e2e = {"value": e / (pipe_ms * 1e-3), "unit": UNIT, "ms_per_step": pipe_ms,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "api": "GeeEncoder.run_host_async (pinned host edge list in, pinned host Z out, "
                      "double-buffered: step i's D2H overlaps step i+1's H2D)",
               "serial": {"value": e / (serial_ms * 1e-3), "ms_per_step": serial_ms,
                          "api": "GeeEncoder.run_host (copies in, pipeline, copy out; one step at a time)"},
               "device_error_bits": _device_err2}

    cpu = None
    if not args.no_cpu_baseline:
        arrays = host_arrays(c)
        times, es = cpu_reference_time(arrays, c, args.cpu_budget_s, 1, 5, sample=args.cpu_sample_edges)
        what = (f"full configs[{args.config}] workload" if es == e else
                f"the first {es} of the {e} edges of configs[{args.config}] (same N, K, options)")
        cpu = {"value": es / statistics.mean(times), "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"{what}, {len(times)} runs of the C restatement (oracle/gee_oracle.c) of "
                         f"encode(EdgeList.to_csr(), ...) on this host ({os.cpu_count()} cores visible, 1 "
                         "used: the reference is single-threaded)",
               "seconds_per_run": statistics.mean(times)}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": (value / PUBLISHED[args.config]) if args.config in PUBLISHED else None,
        "vs_baseline_basis": "PAPER.md:93 sparse GEE 0.6 s for SBM 10k/5.6M edges lap+diag+corr "
                             "(laptop i5) = 9.33e6 edges/s" if args.config in PUBLISHED else None,
        "dtype": "f64" + ("; Z stored f32 (--fp32)" if args.fp32 else ""),
        "data": "synthetic (seeded counter-based generator, BASELINE.json shapes)",
        "config": workload_desc(c),
        "workload_detail": dict(variant=c.get("variant"), l2=((f"flushed: {args.flush_mib} MiB write before every timed step"
                                              + (f", then a {args.flush_mib} MiB read (write-backs drained: cold, "
                                                 "clean L2)" if args.flush_mode == "clean" else ""))
                                             if args.flush_mib > 0 else "not flushed"),
                       stream_entries=m_stream, nnz=nnz,
                       unit_weights=bool(w is None),
                       weights_read_per_step="none: EdgeList found every weight == 1.0 at "
                       "construction, values are implicit" if w is None else "yes"),
        "roofline": roofline,
        "embed_kernel": ({"kernel": emb["kernel"], "ms_per_launch": emb["ms_per_launch"], "gbs": emb["gbs"],
                          "frac": emb["gbs"] / hbm, "alg_bytes_per_launch": emb["alg_bytes"],
                          "traffic": _traffic(args.config, emb["kernel"])} if emb else None),
        # SURVEY 8(d) scope T1: the product kernel alone (inputs resident); the
        # line's value is T2 (device pipeline) and e2e is T3 (host to host)
        "t1": ({"kernel": prod["kernel"], "ms": prod["ms_per_launch"],
                "edges_per_s": e / (prod["ms_per_launch"] * 1e-3),
                "nnz_per_s": nnz / (prod["ms_per_launch"] * 1e-3)} if prod else None),
        "kernels": ktab,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "launch_mode": "eager" if args.eager else "cuda_graph (one graph replay per step)",
        "clocks": sampler.summary(),
        "device_error_bits": _device_err,
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
