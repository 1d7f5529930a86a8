"""Input containers with the reference's names, fields and validation rules.

* EdgeList    -- graph_io.py:48-92  (n_nodes, rows, cols, weights, directed)
* LabelVector -- embedding.py:34-71 (labels in {-1..K-1}, k_classes)
* EmbedOptions-- embedding.py:74-89 (laplacian, diagonal, correlation)

Arrays may be numpy (validated on the host exactly like the reference, same
messages) or CUDA tensors (validated on the device by gee_validate_edges /
the label kernel).  Weights keep float32 when given float32: the reference
promotes them to float64 (graph_io.py:61), which is exact, so the device path
reads the 4-byte values and widens in registers.  ``weights=None`` means
every weight is 1.0 and no weight array is read at all.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib
from .errors import StructuralError

UNLABELED = -1


def _is_tensor(x) -> bool:
    return isinstance(x, torch.Tensor)


class EdgeList:
    """Raw (i, j, weight) triplets plus the node universe they live in."""

    def __init__(self, n_nodes: int, rows=None, cols=None, weights=None, directed: bool = False,
                 *, validate: bool = True):
        self.n_nodes = int(n_nodes)
        self.directed = bool(directed)
        if rows is None:
            rows = np.empty(0, np.int64)
        if cols is None:
            cols = np.empty(0, np.int64)
        on_dev = _is_tensor(rows) and rows.is_cuda
        if on_dev:
            dev = rows.device
            self.rows = rows.to(torch.int64).contiguous()
            self.cols = _device.to_device(cols, torch.int64, dev)
            if weights is None:
                self.weights = None
            else:
                wt = weights if _is_tensor(weights) else torch.as_tensor(np.asarray(weights))
                wdt = torch.float32 if wt.dtype == torch.float32 else torch.float64
                self.weights = _device.to_device(wt, wdt, dev)
        else:
            self.rows = np.ascontiguousarray(rows.cpu().numpy() if _is_tensor(rows) else rows,
                                             dtype=np.int64)
            self.cols = np.ascontiguousarray(cols.cpu().numpy() if _is_tensor(cols) else cols,
                                             dtype=np.int64)
            if weights is None:
                self.weights = None
            else:
                w = weights.cpu().numpy() if _is_tensor(weights) else np.asarray(weights)
                wdt = np.float32 if w.dtype == np.float32 else np.float64
                self.weights = np.ascontiguousarray(w, dtype=wdt)
        n_w = None if self.weights is None else int(self.weights.shape[0])
        if not (self.rows.shape == self.cols.shape) or (n_w is not None and n_w != self.rows.shape[0]):
            raise StructuralError("edge arrays must have equal length")
        # True when every weight is exactly 1.0 (an unweighted graph): the
        # device path then never reads the weight array.  Established by the
        # same construction-time scan that checks finiteness (graph_io.py:71).
        self.unit_weights = self.weights is None
        # True when every weight is >= 0 (established by the same scan; None =
        # not checked).  Lets encode() take the bucketed stream path, whose
        # any-order sums are within 1e-12 only without cancellation.
        self.nonneg = True if self.weights is None else None
        if validate and self.n_edges:
            self._validate()

    def _validate(self):
        # graph_io.py:64-72
        if isinstance(self.rows, torch.Tensor):
            dev = self.rows.device
            err = _device.error_word(dev)
            wt, w = self.weight_kind()
            with torch.cuda.device(dev):
                _lib.check(_lib.load().gee_validate_edges(
                    _device.ptr(self.rows), _device.ptr(self.cols), _device.ptr(w), wt,
                    self.n_edges, self.n_nodes, _device.ptr(err), _device.stream_handle()))
            bits = int(err.item())
            if bits & _lib.ERR_EDGE_RANGE:
                raise StructuralError(f"edge endpoint outside node range [0, {self.n_nodes})")
            if bits & _lib.ERR_EDGE_WEIGHT:
                raise StructuralError("edge weights must be finite")
            if self.weights is not None:
                flags = torch.stack([(self.weights == 1.0).all(), (self.weights >= 0).all()]).cpu()
                self.unit_weights, self.nonneg = bool(flags[0]), bool(flags[1])
            return
        hi = max(int(self.rows.max()), int(self.cols.max()))
        lo = min(int(self.rows.min()), int(self.cols.min()))
        if lo < 0 or hi >= self.n_nodes:
            raise StructuralError(f"edge endpoint outside node range [0, {self.n_nodes})")
        if self.weights is not None:
            if not np.isfinite(self.weights).all():
                raise StructuralError("edge weights must be finite")
            self.unit_weights = bool((self.weights == 1.0).all())
            self.nonneg = bool((self.weights >= 0).all())

    @property
    def n_edges(self) -> int:
        return int(self.rows.shape[0])

    @property
    def on_device(self) -> bool:
        return isinstance(self.rows, torch.Tensor)

    def weight_kind(self):
        """(GEE_W_* code, weight array or None)."""
        if self.weights is None or self.unit_weights:
            return _lib.W_UNIT, None
        dt = self.weights.dtype
        f32 = dt == torch.float32 or dt == np.float32
        return (_lib.W_F32 if f32 else _lib.W_F64), self.weights

    def to_device(self, device=None) -> "EdgeList":
        dev = torch.device(device) if device is not None else _device.require_gpu()
        if self.on_device and self.rows.device == dev:
            return self
        w = None
        if self.weights is not None and not self.unit_weights:
            f32 = self.weights.dtype in (np.float32, torch.float32)
            w = _device.to_device(self.weights, torch.float32 if f32 else torch.float64, dev)
        out = EdgeList(self.n_nodes, _device.to_device(self.rows, torch.int64, dev),
                       _device.to_device(self.cols, torch.int64, dev), w, self.directed,
                       validate=False)
        out.unit_weights = self.unit_weights
        out.nonneg = self.nonneg
        return out

    def weights_f64(self) -> np.ndarray:
        """Host float64 weights as the reference stores them."""
        if self.weights is None:
            return np.ones(self.n_edges)
        w = self.weights.cpu().numpy() if isinstance(self.weights, torch.Tensor) else self.weights
        return np.asarray(w, dtype=np.float64)

    def to_csr(self):
        """Adjacency matrix on the device (graph_io.py:78-92): undirected lists
        are symmetrised, duplicates summed in stream order, zeros dropped."""
        from .sparse import CsrMatrix
        return CsrMatrix.from_edges(self)


class LabelVector:
    """Per-node class assignment in {0..k_classes-1}, or -1 for unlabeled."""

    def __init__(self, labels, k_classes: int):
        self.k_classes = int(k_classes)
        if _is_tensor(labels) and labels.is_cuda:
            self.labels = labels.to(torch.int64).contiguous()  # validated by the K1 kernel
        else:
            lab = labels.cpu().numpy() if _is_tensor(labels) else labels
            self.labels = np.ascontiguousarray(lab, dtype=np.int64)
        if self.k_classes < 1:
            raise StructuralError("k_classes must be at least 1")
        if isinstance(self.labels, np.ndarray) and self.labels.size:
            # embedding.py:45-51
            if self.labels.min() < UNLABELED:
                raise StructuralError("labels below -1 are not allowed")
            if self.labels.max() >= self.k_classes:
                raise StructuralError(
                    f"label {int(self.labels.max())} exceeds k_classes={self.k_classes}")

    def __len__(self) -> int:
        return int(self.labels.shape[0])

    @classmethod
    def from_values(cls, values, k_classes: int | None = None) -> "LabelVector":
        values = np.ascontiguousarray(values, dtype=np.int64)
        if k_classes is None:
            if values.size == 0 or values.max() < 0:
                raise StructuralError("cannot infer class count from labels with no labeled node")
            k_classes = int(values.max()) + 1
        return cls(values, k_classes)

    def class_counts(self) -> np.ndarray:
        """n_k computed by the K1 kernel (bit-exact with embedding.py:68-71)."""
        from .embedding import label_tables
        _, counts, _ = label_tables(self)
        return counts.cpu().numpy()


@dataclass(frozen=True)
class EmbedOptions:
    """Pipeline switches; all 8 combinations are legal."""

    laplacian: bool = False
    diagonal: bool = False
    correlation: bool = False

    @staticmethod
    def all_combinations() -> list["EmbedOptions"]:
        return [EmbedOptions(lap, diag, corr) for lap in (False, True) for diag in (False, True)
                for corr in (False, True)]

    @property
    def flags(self) -> int:
        return ((_lib.LAPLACIAN if self.laplacian else 0) | (_lib.DIAGONAL if self.diagonal else 0)
                | (_lib.CORRELATION if self.correlation else 0))


def options_flags(opts) -> int:
    """Flags of an EmbedOptions-like object (ours or the reference's)."""
    if opts is None:
        return 0
    return ((_lib.LAPLACIAN if opts.laplacian else 0) | (_lib.DIAGONAL if opts.diagonal else 0)
            | (_lib.CORRELATION if opts.correlation else 0))
