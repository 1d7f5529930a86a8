"""The C ABI: libgee.so loads without a GPU and exports exactly what
include/gee.h declares; the ctypes table matches the header."""

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gee.h")
LIB = os.path.join(ROOT, "paper_2406_03726_b200", "libgee.so")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gee_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("gee_label_hist", "gee_csr_build", "gee_degree", "gee_embed", "gee_encode_edges",
                 "gee_add_identity", "gee_laplacian_normalize", "gee_validate_edges"):
        assert must in names


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "build() first"
    lib = ctypes.CDLL(LIB)
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (gee_\w+)", out))
    assert exported == set(declared_functions())


def test_ctypes_table_matches_header():
    from paper_2406_03726_b200 import _lib
    assert set(_lib.SIGNATURES) == set(declared_functions())
    lib = _lib.load()
    assert lib.gee_version().decode().startswith("gee-b200")
    assert lib.gee_status_string(0).decode() == "ok"


def test_size_queries_and_argument_checks_need_no_gpu():
    from paper_2406_03726_b200 import _lib
    lib = _lib.load()
    for wt in (_lib.W_UNIT, _lib.W_F64):
        n = _lib.size_query(lib.gee_encode_edges_workspace, 5_500_000, 10_000, 3, 0, wt)
        assert n > 11_000_000 * 12  # holds at least the 2E-entry CSR
    with pytest.raises(Exception):
        _lib.size_query(lib.gee_encode_edges_workspace, -1, 10, 3, 0, 1)
    out = ctypes.c_size_t(0)
    assert lib.gee_embed_workspace(-5, 10, ctypes.byref(out)) == _lib.GEE_E_ARG


def test_sass_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
