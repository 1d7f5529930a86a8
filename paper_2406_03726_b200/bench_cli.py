"""`bench` / `embed` on the reference's own terms (cli.py:162-241, :97-126):
the same flags, the same CSV schema ``dataset,pipeline,lap,diag,corr,repeat,
seconds`` and table, and a ``--pipeline both`` agreement check at the
reference's PIPELINE_MISMATCH_TOL (1e-12, cli.py:40) -- with GPU pipelines:

* ``gpu``      encode(EdgeList, labels, opts): the fused device pipeline
               (gee_encode_edges), host arrays in, host Z out;
* ``gpu-ops``  encode(edges.to_csr(), labels, opts): the operator seam one
               call at a time (CSR build, then the encode of the CsrMatrix),
               i.e. the reference's own call form (cli.py:176);
* ``sparse``   the reference's name for that call form (same as gpu-ops);
* ``reference`` encode_reference(edges, labels, opts) (cli.py:178,
               embedding.py:146-200);
* ``both``     sparse and reference, compared as cli.py:190-214 does.

Each repeat is timed with time.perf_counter around the call, as
_time_pipeline does (cli.py:170-180); the file parsing stays outside.

    python -m paper_2406_03726_b200.bench_cli bench --edges E --labels L --grid --pipeline both
    python -m paper_2406_03726_b200.bench_cli embed --edges E --labels L --lap --out z.csv
"""

from __future__ import annotations

import argparse
import pathlib
import sys
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import textio as T
from .errors import GpuUnavailableError, NumericalDomainError, ParseError, StructuralError

EXIT_OK, EXIT_INTERNAL, EXIT_USAGE, EXIT_PARSE, EXIT_SHAPE = 0, 1, 2, 3, 4
PIPELINE_MISMATCH_TOL = 1e-12


@dataclass
class BenchResult:
    dataset: str
    pipeline: str
    options: object
    seconds: list = field(default_factory=list)

    @property
    def repeats(self) -> int:
        return len(self.seconds)

    @property
    def mean_s(self) -> float:
        return sum(self.seconds) / len(self.seconds)

    @property
    def min_s(self) -> float:
        return min(self.seconds)


def _bool_flag(token: str) -> bool:
    t = token.strip().lower()
    if t in ("1", "true", "t", "yes", "y", "on"):
        return True
    if t in ("0", "false", "f", "no", "n", "off"):
        return False
    raise argparse.ArgumentTypeError(f"expected a boolean, got {token!r}")


def _tf(flag: bool) -> str:
    return "true" if flag else "false"


def _read_edges(args):
    opts = T.ParseOptions(index_base=1 if args.one_based else 0, directed=args.directed)
    return T.parse_edge_list(pathlib.Path(args.edges), opts, n_nodes=args.nodes)


def _read_labels(args, n_nodes):
    opts = T.ParseOptions(index_base=1 if args.one_based else 0)
    labels = T.parse_labels(pathlib.Path(args.labels), opts, k_classes=args.classes, n_nodes=n_nodes)
    if len(labels) != n_nodes:
        raise StructuralError(f"label file has {len(labels)} entries for {n_nodes} nodes")
    return labels


def _combos(args):
    from .graph import EmbedOptions
    if args.grid:
        return EmbedOptions.all_combinations()
    if args.all_options:
        return [EmbedOptions(laplacian=True, diagonal=True, correlation=True)]
    return [EmbedOptions(laplacian=args.lap, diagonal=args.diag, correlation=args.corr)]


def _time_pipeline(pipeline, edges, labels, opts, repeats):
    from .embedding import encode, encode_reference
    seconds, z = [], None
    for _ in range(repeats):
        t0 = time.perf_counter()
        if pipeline == "gpu":
            z = encode(edges, labels, opts)
        elif pipeline == "reference":  # cli.py:178 encode_reference(edges, ...)
            z = encode_reference(edges, labels, opts)
        else:  # "gpu-ops" / "sparse": encode(edges.to_csr(), ...) (cli.py:176)
            z = encode(edges.to_csr(), labels, opts)
        seconds.append(time.perf_counter() - t0)
    return seconds, np.asarray(z)


def cmd_bench(args) -> int:
    if args.repeats < 1:
        print("error: --repeats must be at least 1", file=sys.stderr)
        return EXIT_USAGE
    edges = _read_edges(args)
    labels = _read_labels(args, edges.n_nodes)
    dataset = Path(args.edges).stem
    # "both" compares the reference's two pipelines as cli.py:190 does
    pipelines = ["sparse", "reference"] if args.pipeline == "both" else [args.pipeline]
    results = []
    # warm-up (library load, workspace, first launches) outside the timed repeats
    _time_pipeline(pipelines[0], edges, labels, _combos(args)[0], 1)
    for opts in _combos(args):
        outputs = {}
        for pipeline in pipelines:
            seconds, z = _time_pipeline(pipeline, edges, labels, opts, args.repeats)
            results.append(BenchResult(dataset, pipeline, opts, seconds))
            outputs[pipeline] = z
        if len(pipelines) == 2:
            delta = outputs[pipelines[0]] - outputs[pipelines[1]]
            diff = float(np.max(np.abs(delta))) if delta.size else 0.0
            print(f"[bench] {dataset} lap={_tf(opts.laplacian)} diag={_tf(opts.diagonal)} "
                  f"corr={_tf(opts.correlation)} max_abs_diff={diff:.3e}", file=sys.stderr)
            if diff > PIPELINE_MISMATCH_TOL:
                print(f"error: pipelines disagree by {diff:.3e} (tolerance {PIPELINE_MISMATCH_TOL:.0e})",
                      file=sys.stderr)
                return EXIT_INTERNAL
    for r in results:
        print(f"[bench] {r.dataset} {r.pipeline} lap={_tf(r.options.laplacian)} diag={_tf(r.options.diagonal)} "
              f"corr={_tf(r.options.correlation)} repeats={r.repeats} mean={r.mean_s:.6f}s min={r.min_s:.6f}s",
              file=sys.stderr)
    if args.format == "csv":
        print("dataset,pipeline,lap,diag,corr,repeat,seconds")
        for r in results:
            for rep, sec in enumerate(r.seconds, start=1):
                print(f"{r.dataset},{r.pipeline},{_tf(r.options.laplacian)},{_tf(r.options.diagonal)},"
                      f"{_tf(r.options.correlation)},{rep},{sec!r}")
    else:
        header = ("dataset", "pipeline", "lap", "diag", "corr", "repeats", "mean_s", "min_s")
        rows = [(r.dataset, r.pipeline, _tf(r.options.laplacian), _tf(r.options.diagonal),
                 _tf(r.options.correlation), str(r.repeats), f"{r.mean_s:.6f}", f"{r.min_s:.6f}") for r in results]
        widths = [max(len(h), *(len(row[i]) for row in rows)) if rows else len(h) for i, h in enumerate(header)]
        print("  ".join(h.ljust(w) for h, w in zip(header, widths)))
        for row in rows:
            print("  ".join(c.ljust(w) for c, w in zip(row, widths)))
    return EXIT_OK


def cmd_embed(args) -> int:
    from .embedding import encode
    from .graph import EmbedOptions
    edges = _read_edges(args)
    labels = _read_labels(args, edges.n_nodes)
    opts = EmbedOptions(laplacian=args.lap, diagonal=args.diag, correlation=args.corr)
    t0 = time.perf_counter()
    z = np.asarray(encode(edges, labels, opts))
    elapsed = time.perf_counter() - t0
    if args.out == "-":
        T.write_embedding(z, sys.stdout)
    else:
        with open(args.out, "w", encoding="utf-8", newline="") as f:
            T.write_embedding(z, f)
    # the reference's summary line (cli.py:115-125): stored entries of the CSR
    # and the undirected edge density 2|E| / (n (n - 1)) of distinct pairs
    nnz = edges.to_csr().nnz
    if edges.n_nodes >= 2:
        density = f"{2.0 * _distinct_pairs(edges) / (edges.n_nodes * (edges.n_nodes - 1.0)):#.5g}"
    else:
        density = "n/a"
    print(f"[embed] nodes={edges.n_nodes} edges={edges.n_edges} classes={labels.k_classes} nnz={nnz} "
          f"density={density} elapsed={elapsed:.6f}s", file=sys.stderr)
    return EXIT_OK


def _distinct_pairs(edges) -> int:
    """Distinct unordered pairs {i, j}, i != j (graph_io.count_undirected_edges), on the device."""
    import torch
    e = edges.to_device()
    lo, hi = torch.minimum(e.rows, e.cols), torch.maximum(e.rows, e.cols)
    keep = lo != hi
    return int(torch.unique(lo[keep] * e.n_nodes + hi[keep]).numel()) if bool(keep.any()) else 0


def build_parser():
    p = argparse.ArgumentParser(prog="gee-b200", description="GEE on B200: embed and bench")
    sub = p.add_subparsers(dest="command", required=True)
    for name in ("embed", "bench"):
        s = sub.add_parser(name)
        s.add_argument("--edges", required=True)
        s.add_argument("--labels", required=True)
        s.add_argument("--classes", type=int)
        s.add_argument("--nodes", type=int)
        s.add_argument("--one-based", action="store_true")
        s.add_argument("--directed", action="store_true")
        if name == "embed":
            s.add_argument("--lap", action="store_true")
            s.add_argument("--diag", action="store_true")
            s.add_argument("--corr", action="store_true")
            s.add_argument("--out", required=True)
            s.set_defaults(func=cmd_embed)
        else:
            s.add_argument("--all-options", action="store_true")
            s.add_argument("--lap", type=_bool_flag, default=False, metavar="B")
            s.add_argument("--diag", type=_bool_flag, default=False, metavar="B")
            s.add_argument("--corr", type=_bool_flag, default=False, metavar="B")
            s.add_argument("--grid", action="store_true")
            s.add_argument("--repeats", type=int, default=5)
            s.add_argument("--pipeline", choices=("gpu", "gpu-ops", "sparse", "reference", "both"), default="gpu")
            s.add_argument("--format", choices=("csv", "table"), default="csv")
            s.set_defaults(func=cmd_bench)
    return p


def main(argv=None) -> int:
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as exc:  # cli.py:333-336: usage errors exit 2, --help 0
        return EXIT_USAGE if exc.code else EXIT_OK
    try:
        return args.func(args)
    except ParseError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_PARSE
    except (StructuralError, NumericalDomainError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_SHAPE
    except OSError as e:  # cli.py:343-345
        print(f"error: {e}", file=sys.stderr)
        return EXIT_PARSE
    except GpuUnavailableError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INTERNAL


if __name__ == "__main__":
    sys.exit(main())
