"""Text formats of the reference (graph_io.py:1-15, :95-305): edge-list and
label parsers, the byte-exact embedding CSV writer, and the edge-list / label
writers.  Host-side I/O around the device path -- parsing and writing are
outside the reference's timed region (cli.py:170-180) -- restated from the
reference's documented behaviour:

* data lines: stripped; blank lines and lines starting with ``#`` skipped
  (graph_io.py:95-100); the delimiter is pinned or auto-detected from the
  FIRST data line (comma if it holds one, else whitespace; :108-111); comma
  fields are stripped (:103-106);
* indices are Python ``int()`` tokens, rejected below the index base and
  shifted by it (:114-121); weights are ``float()`` tokens that must be
  finite (:146-152); a 2-field line takes ``default_weight``;
* the node count is the declared one (indices beyond it rejected) or
  max index + 1 (:153-173);
* labels: one per line, or ``node label`` pairs (form fixed by the first
  data line; unmentioned nodes -1; conflicting duplicates and labels below
  -1 rejected; :176-257);
* embedding CSV: one row per node, values as the shortest round-trip
  decimal (``repr``), integral values below 1e16 printed bare (:281-292).

Every error is a ParseError carrying the 1-based line number, as the
reference raises (errors.py).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Iterable, TextIO

import numpy as np

from .errors import ParseError, StructuralError
from .graph import EdgeList, LabelVector

UNLABELED = -1
_COMMENT_PREFIX = "#"


@dataclass
class ParseOptions:
    """Knobs for the text parsers (graph_io.py:32-45)."""

    delimiter: str = "auto"  # "auto" | "whitespace" | "comma"
    index_base: int = 0
    directed: bool = False
    default_weight: float = 1.0

    def __post_init__(self):
        if self.delimiter not in ("auto", "whitespace", "comma"):
            raise StructuralError(f"unknown delimiter mode {self.delimiter!r}")
        if self.index_base not in (0, 1):
            raise StructuralError("index_base must be 0 or 1")


def _lines(source):
    if isinstance(source, str):
        source = source.splitlines()
    for line_no, raw in enumerate(source, start=1):
        line = raw.strip()
        if line and not line.startswith(_COMMENT_PREFIX):
            yield line_no, line


def _fields(line: str, delimiter: str) -> list[str]:
    if delimiter == "comma":
        return [t.strip() for t in line.split(",")]
    return line.split()


def _index(token: str, base: int, line_no: int, what: str) -> int:
    try:
        value = int(token)
    except ValueError:
        raise ParseError(f"bad {what} {token!r}", line_no) from None
    if value < base:
        raise ParseError(f"{what} {value} below index base {base}", line_no)
    return value - base


def _delimiter(first: str, opts: ParseOptions) -> str:
    if opts.delimiter != "auto":
        return opts.delimiter
    return "comma" if "," in first else "whitespace"


def parse_edge_list(source: Iterable[str] | str, opts: ParseOptions | None = None,
                    n_nodes: int | None = None) -> EdgeList:
    """Edge-list text -> EdgeList (int64 rows/cols, float64 weights)."""
    opts = opts or ParseOptions()
    delim = None
    rows, cols, weights = [], [], []
    top = -1
    for line_no, line in _lines(source):
        if delim is None:
            delim = _delimiter(line, opts)
        f = _fields(line, delim)
        if len(f) not in (2, 3):
            raise ParseError(f"expected 'i j' or 'i j w', got {len(f)} fields", line_no)
        i = _index(f[0], opts.index_base, line_no, "node index")
        j = _index(f[1], opts.index_base, line_no, "node index")
        if len(f) == 3:
            try:
                w = float(f[2])
            except ValueError:
                raise ParseError(f"bad edge weight {f[2]!r}", line_no) from None
            if not math.isfinite(w):
                raise ParseError(f"non-finite edge weight {f[2]!r}", line_no)
        else:
            w = opts.default_weight
        hi = i if i > j else j
        if n_nodes is not None and hi >= n_nodes:
            raise ParseError(f"node index {hi} outside declared node count {n_nodes}", line_no)
        rows.append(i)
        cols.append(j)
        weights.append(w)
        top = max(top, hi)
    count = n_nodes if n_nodes is not None else top + 1
    return EdgeList(count, np.asarray(rows, dtype=np.int64), np.asarray(cols, dtype=np.int64),
                    np.asarray(weights, dtype=np.float64), directed=opts.directed)


def _label(token: str, line_no: int) -> int:
    try:
        value = int(token)
    except ValueError:
        raise ParseError(f"bad label {token!r}", line_no) from None
    if value < UNLABELED:
        raise ParseError(f"label {value} below -1", line_no)
    return value


def parse_labels(source: Iterable[str] | str, opts: ParseOptions | None = None, k_classes: int | None = None,
                 n_nodes: int | None = None) -> LabelVector:
    """Label text (per-line or ``node label`` pairs) -> LabelVector."""
    opts = opts or ParseOptions()
    delim = None
    pairs = None
    seq: list[int] = []
    assigned: dict[int, int] = {}
    top = -1
    for line_no, line in _lines(source):
        if delim is None:
            delim = _delimiter(line, opts)
        f = _fields(line, delim)
        if pairs is None:
            if len(f) == 1:
                pairs = False
            elif len(f) == 2:
                pairs = True
            else:
                raise ParseError(f"expected 'label' or 'node label', got {len(f)} fields", line_no)
        if pairs:
            if len(f) != 2:
                raise ParseError(f"expected 'node label', got {len(f)} fields", line_no)
            node = _index(f[0], opts.index_base, line_no, "node index")
            lab = _label(f[1], line_no)
            if n_nodes is not None and node >= n_nodes:
                raise ParseError(f"node index {node} outside declared node count {n_nodes}", line_no)
            if node in assigned and assigned[node] != lab:
                raise ParseError(f"conflicting labels {assigned[node]} and {lab} for node {node}", line_no)
            assigned[node] = lab
            top = max(top, node)
        else:
            if len(f) != 1:
                raise ParseError(f"expected a single label, got {len(f)} fields", line_no)
            seq.append(_label(f[0], line_no))
    if pairs:
        values = np.full(n_nodes if n_nodes is not None else top + 1, UNLABELED, dtype=np.int64)
        for node, lab in assigned.items():
            values[node] = lab
    else:
        values = np.asarray(seq, dtype=np.int64)
    return LabelVector.from_values(values, k_classes)


def format_value(v: float) -> str:
    """Shortest round-trip decimal; integral values below 1e16 print bare."""
    v = float(v)
    if math.isfinite(v) and v == int(v) and abs(v) < 1e16:
        return str(int(v))
    return repr(v)


def write_embedding(z, sink: TextIO) -> None:
    """Z as CSV, one node per row, K columns (byte-identical to the
    reference's writer)."""
    for row in np.asarray(z):
        sink.write(",".join(format_value(v) for v in row))
        sink.write("\n")


def write_edge_list(edges: EdgeList, sink: TextIO) -> None:
    """``i j w`` lines; parsing them back reproduces the triplets."""
    w = edges.weights if edges.weights is not None else np.ones(edges.n_edges)
    for i, j, x in zip(np.asarray(edges.rows), np.asarray(edges.cols), np.asarray(w)):
        sink.write(f"{i} {j} {format_value(x)}\n")


def write_labels(labels: LabelVector, sink: TextIO) -> None:
    """One label per line (line number = node id)."""
    for lab in np.asarray(labels.labels):
        sink.write(f"{lab}\n")
