"""Loader for tests/golden/reference_cases.npz (made by tests/golden/make_golden.py
from the reference package itself)."""

import functools
import os

import numpy as np

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_cases.npz")
COMBOS = [(lap, diag, corr) for lap in (0, 1) for diag in (0, 1) for corr in (0, 1)]


@functools.lru_cache(maxsize=1)
def load():
    data = np.load(PATH, allow_pickle=False)
    store = {k: data[k] for k in data.files}
    out = []
    for idx, name in enumerate(store["names"]):
        p = f"c{idx}_"
        case = {k[len(p):]: v for k, v in store.items() if k.startswith(p)}
        n, k, directed = (int(x) for x in case["meta"])
        case.update(name=str(name), n=n, k=k, directed=bool(directed))
        out.append(case)
    return out


def ztag(lap, diag, corr):
    return f"z{lap}{diag}{corr}"


EXTRA_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_extra.npz")


@functools.lru_cache(maxsize=1)
def load_extra():
    """tests/golden/reference_extra.npz (make_extra_golden.py): W, encode_reference
    and from_triplets of the reference on the same seeded inputs."""
    data = np.load(EXTRA_PATH, allow_pickle=False)
    store = {k: data[k] for k in data.files}
    out = []
    for idx, name in enumerate(store["names"]):
        p = f"c{idx}_"
        case = {k[len(p):]: v for k, v in store.items() if k.startswith(p)}
        n, k, directed = (int(x) for x in case["meta"])
        case.update(name=str(name), n=n, k=k, directed=bool(directed))
        out.append(case)
    return out


def rtag(lap, diag, corr):
    return f"r{lap}{diag}{corr}"
