"""ctypes binding of libgee.so (include/gee.h) -- the only compute path.

There is no CPU fallback: importing the ops without the built library, or
calling them without a CUDA device, raises immediately.
"""

from __future__ import annotations

import ctypes
import os

from .errors import GpuUnavailableError, NumericalDomainError, StructuralError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgee.so")

# synchronous status codes / device error bits / option flags (gee.h)
GEE_OK, GEE_E_ARG, GEE_E_WORKSPACE, GEE_E_CUDA = 0, 1, 2, 3
ERR_NEG_DEGREE, ERR_NONFINITE, ERR_LABEL, ERR_EDGE_RANGE, ERR_EDGE_WEIGHT = 1, 2, 4, 8, 16
ERR_NEG_WEIGHT = 32
LAPLACIAN, DIAGONAL, CORRELATION = 1, 2, 4
NONNEG, FP32 = 8, 16  # caller asserts weights >= 0 (stream path) / float32 Z
W_UNIT, W_F64, W_F32 = 0, 1, 2

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_int = ctypes.c_int
_u32 = ctypes.c_uint
_szp = ctypes.POINTER(ctypes.c_size_t)

# name -> (restype, argtypes); mirrors include/gee.h one to one
SIGNATURES = {
    "gee_version": (ctypes.c_char_p, []),
    "gee_status_string": (ctypes.c_char_p, [_int]),
    "gee_last_error_string": (ctypes.c_char_p, []),
    "gee_validate_edges": (_int, [_vp, _vp, _vp, _int, _i64, _i64, _vp, _vp]),
    "gee_label_hist": (_int, [_vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp]),
    "gee_inv_counts": (_int, [_vp, _i32, _vp, _vp]),
    "gee_weight_matrix_workspace": (_int, [_i64, _szp]),
    "gee_weight_matrix": (_int, [_vp, _i64, _vp, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp]),
    "gee_csr_build_workspace": (_int, [_i64, _i64, _i64, _int, _szp]),
    "gee_csr_build": (_int, [_vp, _vp, _vp, _int, _i64, _i64, _i64, _int, _int, _vp, _vp, _vp, _vp,
                             _vp, _u32, _vp, _vp, _vp, ctypes.c_size_t, _vp, _vp]),
    "gee_degree": (_int, [_vp, _vp, _vp, _i64, _u32, _vp, _vp, _vp, _vp]),
    "gee_add_identity_workspace": (_int, [_i64, _szp]),
    "gee_add_identity": (_int, [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp]),
    "gee_laplacian_normalize_workspace": (_int, [_i64, _szp]),
    "gee_laplacian_normalize": (_int, [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp,
                                       ctypes.c_size_t, _vp, _vp]),
    "gee_embed_workspace": (_int, [_i64, _i64, _szp]),
    "gee_embed": (_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp, _i32, _u32, _vp, _i64,
                         _vp, ctypes.c_size_t, _vp, _vp]),
    "gee_encode_edges_workspace": (_int, [_i64, _i64, _i32, _int, _int, _szp]),
    "gee_encode_edges": (_int, [_vp, _vp, _vp, _int, _i64, _i64, _int, _vp, _i32, _u32, _vp, _vp,
                                ctypes.c_size_t, _vp, _vp]),
    "gee_bitmap_shard_workspace": (_int, [_i64, _i64, _i64, _i64, _i32, _szp]),
    "gee_bitmap_shard_degrees": (_int, [_vp, _vp, _i64, _i64, _i64, _i64, _vp, _i32, _u32, _vp, _vp,
                                        ctypes.c_size_t, _vp, _vp]),
    "gee_bitmap_shard_encode": (_int, [_vp, _vp, _i64, _i64, _i64, _i64, _i32, _u32, _vp, _vp, _vp,
                                       ctypes.c_size_t, _vp, _vp]),
    "gee_shuffle_buckets": (_i64, [_i64]),
    "gee_shuffle_row_hist": (_int, [_vp, _vp, _i64, _i64, _int, _vp, _vp]),
    "gee_shuffle_bounds": (_int, [_vp, _i64, _int, _vp, _vp]),
    "gee_partition_workspace": (_int, [_i64, _int, _szp]),
    "gee_partition": (_int, [_vp, _vp, _vp, _int, _i64, _int, _vp, _int, _vp, _vp, _vp, _vp, _vp,
                             ctypes.c_size_t, _vp]),
    "gee_gen_rmat": (_int, [ctypes.c_uint64, ctypes.c_uint64, _int, _i64, _u32, _u32, _u32, _vp, _vp, _vp, _vp]),
    "gee_gen_chunglu": (_int, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _vp, _i64, _i64, _vp, _vp, _vp,
                               _vp]),
    "gee_gen_pairs": (_int, [ctypes.c_uint64, _i64, _i64, _i64, _vp, _vp]),
    "gee_gen_sbm_count": (_int, [ctypes.c_uint64, _i64, _vp, _u32, _u32, _vp, _vp]),
    "gee_gen_sbm_fill": (_int, [ctypes.c_uint64, _i64, _vp, _u32, _u32, _vp, _vp, _vp, _vp]),
    "gee_text_workspace": (_int, [_i64, _i64, _szp]),
    "gee_text_count_lines": (_int, [_vp, _i64, _vp, _vp, ctypes.c_size_t, _vp]),
    "gee_parse_edges": (_int, [_vp, _i64, _i64, _int, _int, ctypes.c_double, _i64, _vp, _vp, _vp, _vp, _vp, _vp,
                               _vp, _vp, ctypes.c_size_t, _vp]),
    "gee_parse_labels": (_int, [_vp, _i64, _i64, _int, _int, _i64, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_size_t,
                                _vp]),
    "gee_labels_assign": (_int, [_vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp]),
    "gee_stream_shard_workspace": (_int, [_i64, _i64, _i64, _i64, _i32, _int, _u32, _szp]),
    "gee_stream_shard_degrees": (_int, [_vp, _vp, _vp, _int, _i64, _i64, _i64, _i64, _vp, _i32, _u32, _vp, _vp,
                                        ctypes.c_size_t, _vp, _vp]),
    "gee_stream_shard_encode": (_int, [_int, _i64, _i64, _i64, _i64, _i32, _u32, _vp, _vp, _vp, ctypes.c_size_t,
                                       _vp, _vp]),
    "gee_launch_count": (ctypes.c_uint64, []),
    "gee_reset_launch_count": (None, []),
    "gee_profile_start": (_int, [_vp]),
    "gee_profile_stop": (_int, []),
    "gee_profile_read": (_int, [ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_char_p), _int]),
    "gee_debug_set": (_int, [_int, _int]),
}
DEBUG_FORCE_BUCKETS = 1  # key; values: 0 default, 1 row buckets, 2 no bitmap path, 3 = 2 + 64-bit sort keys
DEBUG_EMBED_FLAT_BYTES = 2  # key; per-warp shared bytes of the K > 8 flat embed blocks (0 = warp per row)
DEBUG_EMBED_FLAT_ROWMAX = 3  # key; longest row a flat embed block takes (longer: a warp each)
DEBUG_STREAM_TILE = 5  # key; KB of the stream encode's Z tile (default 104)
DEBUG_STREAM = 4  # key; bucketed stream encode: 0 auto, 1 never (forces the CSR paths)

_lib = None


def load():
    """Load libgee.so and bind every entry point; raises if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise GpuUnavailableError(
                f"{LIB_PATH} is not built; run __graft_entry__.build() "
                "(make -C paper_2406_03726_b200/csrc)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(status: int):
    """Raise for a synchronous status from the library."""
    if status == GEE_OK:
        return
    lib = load()
    msg = lib.gee_status_string(status).decode()
    if status == GEE_E_CUDA:
        msg += ": " + lib.gee_last_error_string().decode()
    if status == GEE_E_ARG:
        raise StructuralError(f"libgee: {msg}")
    raise RuntimeError(f"libgee: {msg}")


def raise_device_errors(bits: int, context: str = ""):
    """Map device error bits to the reference's exception classes."""
    if not bits:
        return
    where = f" ({context})" if context else ""
    if bits & ERR_EDGE_RANGE:
        raise StructuralError(f"edge endpoint outside node range{where}")
    if bits & ERR_EDGE_WEIGHT:
        raise StructuralError(f"edge weights must be finite{where}")
    if bits & ERR_LABEL:
        raise StructuralError(f"labels must lie in [-1, k_classes){where}")
    if bits & ERR_NEG_DEGREE:
        raise NumericalDomainError(f"negative degree under Laplacian normalization{where}")
    if bits & ERR_NONFINITE:
        raise NumericalDomainError(f"non-finite embedding values{where}")
    if bits & ERR_NEG_WEIGHT:
        raise StructuralError(f"negative edge weight under the non-negative assertion{where}")
    raise RuntimeError(f"libgee device error bits {bits:#x}{where}")


def size_query(fn, *args) -> int:
    out = ctypes.c_size_t(0)
    check(fn(*args, ctypes.byref(out)))
    return int(out.value)
