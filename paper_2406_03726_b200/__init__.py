"""B200-native sparse Graph Encoder Embedding (arXiv 2406.03726).

A drop-in for the reference package's embedding path (pkg/src/graphee):
same names (EdgeList, LabelVector, EmbedOptions, CsrMatrix, encode,
add_identity, degree_vector, laplacian_normalize, the error classes), same
semantics, computed by hand-written sm_100a CUDA kernels in libgee.so
(C ABI: include/gee.h).  There is no CPU fallback.
"""

from .embedding import GeeEncoder, build_weight_matrix, encode, encode_reference, label_tables, spmm_weight
from .errors import GpuUnavailableError, GrapheeError, NumericalDomainError, ParseError, StructuralError
from .graph import UNLABELED, EdgeList, EmbedOptions, LabelVector
from .sparse import CsrMatrix, add_identity, degree_vector, laplacian_normalize

__version__ = "0.1.0"

__all__ = [
    "UNLABELED",
    "CsrMatrix",
    "EdgeList",
    "EmbedOptions",
    "GeeEncoder",
    "GpuUnavailableError",
    "GrapheeError",
    "LabelVector",
    "NumericalDomainError",
    "ParseError",
    "StructuralError",
    "add_identity",
    "build_weight_matrix",
    "degree_vector",
    "encode",
    "encode_reference",
    "label_tables",
    "laplacian_normalize",
    "spmm_weight",
    "__version__",
]
