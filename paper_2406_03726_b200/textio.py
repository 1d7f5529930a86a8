"""Edge-list / label text input on the device, and the embedding CSV writer.

Mirrors the reference's graph_io text interface (graph_io.py:32-45
ParseOptions, :124-173 parse_edge_list, :176-247 parse_labels, :281-305 the
writers) with the parsing itself done by libgee (csrc/k_text.cu): the file's
bytes go to the GPU once, every line is indexed, classified and parsed in
parallel, and the edge arrays come back already on the device (ready for
encode()).  The host only formats the ParseError of the first failing line
(re-reading that one line) and converts the rare weight tokens the device
flags as undecidable (more than 19 significant digits).

Writers stay on the host: the CSV holds each value as its shortest
round-trip decimal (Python repr), integral values below 1e16 bare -- the
byte format of the reference's writer (test_cli.py:10).
"""

from __future__ import annotations

import io
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib
from .errors import ParseError, StructuralError
from .graph import EdgeList, LabelVector

_DELIM = {"auto": 0, "whitespace": 1, "comma": 2}


@dataclass
class ParseOptions:
    """Parser switches with the reference's names and defaults (graph_io.py:32-45)."""

    delimiter: str = "auto"
    index_base: int = 0
    directed: bool = False
    default_weight: float = 1.0

    def __post_init__(self):
        if self.delimiter not in _DELIM:
            raise StructuralError(f"unknown delimiter mode {self.delimiter!r}")
        if self.index_base not in (0, 1):
            raise StructuralError("index_base must be 0 or 1")


def _read_bytes(source) -> bytes:
    """str (the text itself), bytes, a path-like, an open file, or an
    iterable of lines -> the raw text bytes."""
    if isinstance(source, (bytes, bytearray, memoryview)):
        return bytes(source)
    if isinstance(source, str):
        return source.encode()
    if isinstance(source, os.PathLike):
        with open(source, "rb") as f:
            return f.read()
    if isinstance(source, io.TextIOBase) or hasattr(source, "read"):
        data = source.read()
        return data.encode() if isinstance(data, str) else bytes(data)
    # iterable of lines (each keeps or lacks its terminator, like file iteration)
    parts = []
    for line in source:
        s = line if isinstance(line, str) else line.decode()
        parts.append(s if s.endswith(("\n", "\r")) else s + "\n")
    return "".join(parts).encode()


class _Text:
    """The text on the device plus its line index (one H2D copy)."""

    def __init__(self, data: bytes, dev):
        self.data = data
        self.dev = dev
        lib = _lib.load()
        self.nbytes = len(data)
        host = torch.frombuffer(bytearray(data), dtype=torch.uint8) if data else torch.empty(0, dtype=torch.uint8)
        self.buf = host.to(dev)
        nb = _lib.size_query(lib.gee_text_workspace, self.nbytes, 0)
        ws = _device.WORKSPACE.get(nb, dev)
        breaks = torch.zeros(1, dtype=torch.int64, device=dev)
        with torch.cuda.device(dev):
            _lib.check(lib.gee_text_count_lines(_device.ptr(self.buf), self.nbytes, _device.ptr(breaks),
                                                _device.ptr(ws), ws.numel(), _device.stream_handle()))
        self.n_lines = int(breaks.item()) + 1
        nb = _lib.size_query(lib.gee_text_workspace, self.nbytes, self.n_lines)
        self.ws = _device.WORKSPACE.get(nb, dev)
        self.line_start = torch.empty(self.n_lines, dtype=torch.int64, device=dev)

    def line(self, k: int) -> str:
        """Text of line k (0-based), for error messages."""
        ls = self.line_start.cpu().numpy() if not hasattr(self, "_ls") else self._ls
        self._ls = ls
        end = int(ls[k + 1]) if k + 1 < self.n_lines else self.nbytes
        return self.data[int(ls[k]):end].decode(errors="replace")

    def delimiter(self, opts: ParseOptions, first_line: int) -> str:
        if opts.delimiter != "auto":
            return opts.delimiter
        return "comma" if first_line >= 0 and "," in self.line(first_line) else "whitespace"


def _fields(line: str, delim: str) -> list[str]:
    line = line.strip()
    if delim == "comma":
        return [t.strip() for t in line.split(",")]
    return line.split()


# error codes of k_text.cu -> the reference's messages (graph_io.py:124-257)
def _edge_error(text: _Text, word: int, opts: ParseOptions, n_nodes, first_line: int) -> ParseError:
    line_no, code = word >> 8, word & 0xFF
    f = _fields(text.line(line_no - 1), text.delimiter(opts, first_line))
    base = opts.index_base
    if code == 1:
        return ParseError(f"expected 'i j' or 'i j w', got {len(f)} fields", line_no)
    if code in (2, 4):
        return ParseError(f"bad node index {f[0 if code == 2 else 1]!r}", line_no)
    if code in (3, 5):
        v = int(f[0 if code == 3 else 1])
        return ParseError(f"node index {v} below index base {base}", line_no)
    if code == 6:
        return ParseError(f"bad edge weight {f[2]!r}", line_no)
    if code == 7:
        return ParseError(f"non-finite edge weight {f[2]!r}", line_no)
    if code == 8:
        hi = max(int(f[0]), int(f[1])) - base
        return ParseError(f"node index {hi} outside declared node count {n_nodes}", line_no)
    return ParseError(f"malformed line (code {code})", line_no)


def _label_error(text: _Text, word: int, opts: ParseOptions, n_nodes, first_line: int, conflict=None) -> ParseError:
    line_no, code = word >> 8, word & 0xFF
    f = _fields(text.line(line_no - 1), text.delimiter(opts, first_line))
    if code == 1:
        return ParseError(f"expected 'label' or 'node label', got {len(f)} fields", line_no)
    if code == 11:
        return ParseError(f"expected 'node label', got {len(f)} fields", line_no)
    if code == 12:
        return ParseError(f"expected a single label, got {len(f)} fields", line_no)
    if code == 2:
        return ParseError(f"bad node index {f[0]!r}", line_no)
    if code == 3:
        return ParseError(f"node index {int(f[0])} below index base {opts.index_base}", line_no)
    if code == 9:
        return ParseError(f"bad label {f[-1]!r}", line_no)
    if code == 10:
        return ParseError(f"label {int(f[-1])} below -1", line_no)
    if code == 8:
        return ParseError(f"node index {int(f[0]) - opts.index_base} outside declared node count {n_nodes}",
                          line_no)
    if code == 13:
        node = int(f[0]) - opts.index_base
        return ParseError(f"conflicting labels {conflict(node)} and {int(f[1])} for node {node}", line_no)
    return ParseError(f"malformed line (code {code})", line_no)


def parse_edge_list(source, opts: ParseOptions | None = None, n_nodes: int | None = None,
                    device=None) -> EdgeList:
    """Edge-list text -> EdgeList on the device (int64 rows/cols, float64 weights)."""
    opts = opts or ParseOptions()
    dev = torch.device(device) if device is not None else _device.require_gpu()
    data = _read_bytes(source)
    if not data.strip():
        return EdgeList(n_nodes if n_nodes is not None else 0, np.empty(0, np.int64), np.empty(0, np.int64),
                        np.empty(0), directed=opts.directed)
    text = _Text(data, dev)
    m = text.n_lines
    rows = torch.empty(m, dtype=torch.int64, device=dev)
    cols = torch.empty(m, dtype=torch.int64, device=dev)
    w = torch.empty(m, dtype=torch.float64, device=dev)
    fb = torch.empty(m, dtype=torch.uint8, device=dev)
    slot_line = torch.empty(m, dtype=torch.int64, device=dev)
    info = torch.empty(6, dtype=torch.int64, device=dev)
    lib = _lib.load()
    with torch.cuda.device(dev):
        _lib.check(lib.gee_parse_edges(
            _device.ptr(text.buf), text.nbytes, m, _DELIM[opts.delimiter], opts.index_base,
            float(opts.default_weight), -1 if n_nodes is None else int(n_nodes), _device.ptr(text.line_start),
            _device.ptr(rows), _device.ptr(cols), _device.ptr(w), _device.ptr(fb), _device.ptr(slot_line),
            _device.ptr(info), _device.ptr(text.ws), text.ws.numel(), _device.stream_handle()))
    n_edges, top, err, n_fb, first = (int(x) for x in info[:5].cpu())
    if err != -1:
        raise _edge_error(text, err, opts, n_nodes, first)
    rows, cols, w, fb = rows[:n_edges], cols[:n_edges], w[:n_edges], fb[:n_edges]
    if n_fb:
        # > 19 significant digits: Python's float() decides (slots in file order)
        slots = torch.nonzero(fb).flatten()
        data_lines = slot_line[slots].cpu().numpy().tolist()
        slots = slots.cpu().numpy()
        delim = text.delimiter(opts, first)
        vals = []
        for slot, k in zip(slots, data_lines):
            tok = _fields(text.line(k), delim)[2]
            v = float(tok)
            if not math.isfinite(v):
                raise ParseError(f"non-finite edge weight {tok!r}", k + 1)
            vals.append(v)
        w[torch.as_tensor(slots, device=dev)] = torch.as_tensor(vals, dtype=torch.float64, device=dev)
    count = n_nodes if n_nodes is not None else top + 1
    return EdgeList(count, rows, cols, w, directed=opts.directed)


def parse_labels(source, opts: ParseOptions | None = None, k_classes: int | None = None,
                 n_nodes: int | None = None, device=None) -> LabelVector:
    """Label text (one label per line, or ``node label`` pairs) -> LabelVector."""
    opts = opts or ParseOptions()
    dev = torch.device(device) if device is not None else _device.require_gpu()
    data = _read_bytes(source)
    if not data.strip():
        return LabelVector.from_values(np.empty(0, np.int64), k_classes)
    text = _Text(data, dev)
    m = text.n_lines
    node = torch.empty(m, dtype=torch.int64, device=dev)
    lab = torch.empty(m, dtype=torch.int64, device=dev)
    slot_line = torch.empty(m, dtype=torch.int64, device=dev)
    info = torch.empty(6, dtype=torch.int64, device=dev)
    lib = _lib.load()
    with torch.cuda.device(dev):
        _lib.check(lib.gee_parse_labels(
            _device.ptr(text.buf), text.nbytes, m, _DELIM[opts.delimiter], opts.index_base,
            -1 if n_nodes is None else int(n_nodes), _device.ptr(text.line_start), _device.ptr(node),
            _device.ptr(lab), _device.ptr(slot_line), _device.ptr(info), _device.ptr(text.ws), text.ws.numel(),
            _device.stream_handle()))
    n_data, top, err, _, first = (int(x) for x in info[:5].cpu())
    node, lab = node[:n_data], lab[:n_data]
    pairs = n_data > 0 and len(_fields(text.line(first), text.delimiter(opts, first))) == 2
    if not pairs:
        if err != -1:
            raise _label_error(text, err, opts, n_nodes, first)
        return LabelVector.from_values(lab.cpu().numpy(), k_classes)
    size = n_nodes if n_nodes is not None else top + 1
    values = torch.empty(max(size, 0), dtype=torch.int64, device=dev)
    firsts = torch.empty(max(size, 1), dtype=torch.int64, device=dev)
    conflict = torch.full((1,), -1, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        _lib.check(lib.gee_labels_assign(
            _device.ptr(node), _device.ptr(lab), _device.ptr(slot_line), n_data, max(size, 0),
            _device.ptr(firsts), _device.ptr(values), _device.ptr(conflict), _device.stream_handle()))
    cw = int(conflict.item())
    words = [x for x in (err, cw) if x != -1]
    if words:
        vals = values.cpu().numpy()
        raise _label_error(text, min(words), opts, n_nodes, first, conflict=lambda v: int(vals[v]))
    return LabelVector.from_values(values.cpu().numpy(), k_classes)


# ---- writers (host) -----------------------------------------------------------
def _fmt(v: float) -> str:
    """Shortest round-trip decimal; an integral value under 1e16 prints as an int."""
    if v.is_integer() and abs(v) < 1e16:
        return "%d" % v
    return repr(v)


def write_embedding(z, sink) -> None:
    """Z as CSV: one node per line, K comma-separated values."""
    arr = z.cpu().numpy() if isinstance(z, torch.Tensor) else np.asarray(z)
    rows = [",".join(map(_fmt, map(float, r))) for r in arr]
    sink.write("".join(r + "\n" for r in rows))


def write_edge_list(edges: EdgeList, sink) -> None:
    """``i j w`` per line (parsed back to the same triplets)."""
    r = np.asarray(edges.rows.cpu() if isinstance(edges.rows, torch.Tensor) else edges.rows)
    c = np.asarray(edges.cols.cpu() if isinstance(edges.cols, torch.Tensor) else edges.cols)
    w = np.ones(r.size) if edges.weights is None else np.asarray(
        edges.weights.cpu() if isinstance(edges.weights, torch.Tensor) else edges.weights, dtype=np.float64)
    sink.write("".join(f"{a} {b} {_fmt(float(x))}\n" for a, b, x in zip(r.tolist(), c.tolist(), w.tolist())))


def write_labels(labels: LabelVector, sink) -> None:
    """One label per line; line k is node k."""
    lab = labels.labels.cpu().numpy() if isinstance(labels.labels, torch.Tensor) else labels.labels
    sink.write("".join(f"{x}\n" for x in np.asarray(lab).tolist()))
