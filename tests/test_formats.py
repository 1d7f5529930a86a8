"""Text I/O (paper_2406_03726_b200.textio: the device parsers of
csrc/k_text.cu and the host CSV writer) against the reference's own parsers
and writer: tests/golden/formats_cases.json was produced by running
graph_io.py:95-305 itself (tests/golden/make_formats_golden.py)."""

import io
import json
import os

import numpy as np
import pytest

from paper_2406_03726_b200 import errors as E
from paper_2406_03726_b200 import textio as F

CASES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "formats_cases.json")))


def _run(fn):
    try:
        return {"ok": fn()}
    except (E.ParseError, E.StructuralError) as e:
        return {"error": type(e).__name__, "line": getattr(e, "line_no", None)}


def _np(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES["edges"], ids=range(len(CASES["edges"])))
def test_parse_edge_list_matches_reference(case):
    def f():
        e = F.parse_edge_list(io.StringIO(case["text"]), F.ParseOptions(**case["opts"]), n_nodes=case["n_nodes"])
        return {"n_nodes": int(e.n_nodes), "rows": _np(e.rows).tolist(), "cols": _np(e.cols).tolist(),
                "weights": [float(x).hex() for x in _np(e.weights)], "directed": bool(e.directed)}
    assert _run(f) == case["result"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES["labels"], ids=range(len(CASES["labels"])))
def test_parse_labels_matches_reference(case):
    def f():
        lv = F.parse_labels(io.StringIO(case["text"]), F.ParseOptions(**case["opts"]), k_classes=case["k_classes"],
                            n_nodes=case["n_nodes"])
        return {"labels": _np(lv.labels).tolist(), "k_classes": int(lv.k_classes)}
    assert _run(f) == case["result"]


@pytest.mark.parametrize("case", CASES["embedding"], ids=range(len(CASES["embedding"])))
def test_write_embedding_bytes_match_reference(case):
    z = np.array([[float.fromhex(x) for x in row] for row in case["z"]], dtype=np.float64).reshape(-1, case["k"])
    buf = io.StringIO()
    F.write_embedding(z, buf)
    assert buf.getvalue() == case["csv"]


def test_triangle_golden_csv():
    # test_cli.py:10 (GOLDEN_TRIANGLE_CSV)
    buf = io.StringIO()
    F.write_embedding(np.array([[0.0, 1.0], [1.0, 0.5], [1.0, 0.5]]), buf)
    assert buf.getvalue().encode() == b"0,1\n1,0.5\n1,0.5\n"


@pytest.mark.gpu
def test_edge_list_and_labels_round_trip():
    rng = np.random.default_rng(4)
    n, m = 50, 300
    from paper_2406_03726_b200.graph import EdgeList, LabelVector
    e = EdgeList(n, rng.integers(0, n, m), rng.integers(0, n, m), rng.standard_normal(m) * 1e3, directed=True)
    buf = io.StringIO()
    F.write_edge_list(e, buf)
    back = F.parse_edge_list(io.StringIO(buf.getvalue()), F.ParseOptions(directed=True), n_nodes=n)
    assert np.array_equal(_np(back.rows), e.rows) and np.array_equal(_np(back.cols), e.cols)
    assert np.array_equal(_np(back.weights), e.weights)
    lv = LabelVector(rng.integers(-1, 4, n), 4)
    buf = io.StringIO()
    F.write_labels(lv, buf)
    back = F.parse_labels(io.StringIO(buf.getvalue()), k_classes=4)
    assert np.array_equal(_np(back.labels), lv.labels)


def _float_tokens(rng, n):
    """repr() of random doubles across the exponent range, short decimals,
    exponents, underscores, signs, leading zeros and long mantissas."""
    toks = []
    for _ in range(n):
        kind = rng.integers(0, 8)
        if kind == 0:
            toks.append(repr(float(rng.random())))
        elif kind == 1:
            toks.append(repr(float(np.exp(rng.uniform(-700, 700)))))
        elif kind == 2:
            toks.append(f"{rng.integers(0, 10**6)}.{rng.integers(0, 10**4):04d}")
        elif kind == 3:
            toks.append(f"{rng.integers(1, 999)}e{rng.integers(-330, 310)}")
        elif kind == 4:
            toks.append(f"{'-+'[rng.integers(0, 2)]}{rng.integers(0, 10**9)}_{rng.integers(0, 1000):03d}.5")
        elif kind == 5:
            toks.append("0" * int(rng.integers(1, 5)) + repr(float(rng.random() * 1e-5)))
        elif kind == 6:
            toks.append("".join(str(int(d)) for d in rng.integers(0, 10, rng.integers(15, 30))) + "e-10")
        else:
            v = float(rng.integers(1, 2**53)) * 2.0 ** int(rng.integers(-1074, 970))
            toks.append(repr(v) if np.isfinite(v) and v != 0 else "1.5")
    return [t for t in toks if np.isfinite(float(t))]  # inf is a ParseError (tested elsewhere)


@pytest.mark.gpu
def test_device_float_parser_matches_python_float():
    """Every weight token converts to exactly Python's float() (Eisel-Lemire
    on the device, host conversion of the > 19-digit ones)."""
    rng = np.random.default_rng(2024)
    toks = _float_tokens(rng, 20000)
    text = "".join(f"{k % 97} {(k * 7) % 97} {t}\n" for k, t in enumerate(toks))
    e = F.parse_edge_list(text, n_nodes=97)
    got = _np(e.weights)
    want = np.array([float(t) for t in toks])
    bad = np.flatnonzero(got.view(np.int64) != want.view(np.int64))
    assert bad.size == 0, [(toks[i], got[i], want[i]) for i in bad[:5]]


@pytest.mark.gpu
def test_device_parser_line_endings_and_whitespace():
    text = "# header\r\n0\t1  0.25\r\n\r\n  1 2\x0b\r2 3 1e-3\n   \n3 0 7"
    e = F.parse_edge_list(text, F.ParseOptions(delimiter="whitespace"))
    assert _np(e.rows).tolist() == [0, 1, 2, 3] and _np(e.cols).tolist() == [1, 2, 3, 0]
    assert _np(e.weights).tolist() == [0.25, 1.0, 1e-3, 7.0]
    with pytest.raises(E.ParseError) as ex:
        F.parse_edge_list("0 1\n1 2\n3,4\n")  # whitespace from line 1: '3,4' is one field
    assert ex.value.line_no == 3


# ---- the bench / embed harness (bench_cli.py; cli.py:162-241) ----------------
def _files(tmp_path, edges, labels):
    e = tmp_path / "tri_edges.txt"
    lab = tmp_path / "tri_labels.txt"
    e.write_text(edges)
    lab.write_text(labels)
    return str(e), str(lab)


@pytest.mark.gpu
def test_cli_parse_error_exit_code(tmp_path, capsys):
    from paper_2406_03726_b200 import bench_cli
    e, lab = _files(tmp_path, "0 1\n0 x\n", "0\n1\n")
    assert bench_cli.main(["bench", "--edges", e, "--labels", lab]) == bench_cli.EXIT_PARSE
    assert "line 2" in capsys.readouterr().err
    e, lab = _files(tmp_path, "0 1\n1 2\n", "0\n1\n")  # 2 labels for 3 nodes
    assert bench_cli.main(["embed", "--edges", e, "--labels", lab, "--out", "-"]) == bench_cli.EXIT_SHAPE
    assert bench_cli.main(["bench", "--edges", e, "--labels", lab, "--repeats", "0"]) == bench_cli.EXIT_USAGE
    assert bench_cli.main(["embed", "--edges", str(tmp_path / "missing.txt"), "--labels", lab,
                           "--out", "-"]) == bench_cli.EXIT_PARSE  # OSError, cli.py:343-345


def test_cli_usage_exit_codes():
    from paper_2406_03726_b200 import bench_cli
    assert bench_cli.main(["bench"]) == bench_cli.EXIT_USAGE  # missing required flags
    assert bench_cli.main(["--help"]) == bench_cli.EXIT_OK


@pytest.mark.gpu
def test_cli_embed_triangle_golden_bytes(tmp_path):
    from paper_2406_03726_b200 import bench_cli
    e, lab = _files(tmp_path, "0 1\n0 2\n1 2\n", "0\n1\n1\n")
    out = tmp_path / "z.csv"
    assert bench_cli.main(["embed", "--edges", e, "--labels", lab, "--out", str(out)]) == 0
    assert out.read_bytes() == b"0,1\n1,0.5\n1,0.5\n"  # test_cli.py:10


@pytest.mark.gpu
def test_cli_bench_grid_both_pipelines_csv(tmp_path, capsys):
    from paper_2406_03726_b200 import bench_cli
    rng = np.random.default_rng(9)
    n = 400
    r, c = np.nonzero(np.triu(rng.random((n, n)) < 0.05, 1))
    w = 1.0 - rng.random(r.size)
    e, lab = _files(tmp_path, "".join(f"{i} {j} {float(x)!r}\n" for i, j, x in zip(r, c, w)),
                    "".join(f"{x}\n" for x in rng.integers(-1, 4, n)))
    assert bench_cli.main(["bench", "--edges", e, "--labels", lab, "--grid", "--pipeline", "both",
                           "--repeats", "2"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == "dataset,pipeline,lap,diag,corr,repeat,seconds"
    rows = [ln.split(",") for ln in lines[1:]]
    assert len(rows) == 8 * 2 * 2
    assert {x[1] for x in rows} == {"sparse", "reference"} and all(float(x[6]) > 0 for x in rows)
