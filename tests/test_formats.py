"""Text I/O (paper_2406_03726_b200.formats) against the reference's own
parsers and writer: tests/golden/formats_cases.json was produced by running
graph_io.py:95-305 itself (tests/golden/make_formats_golden.py)."""

import io
import json
import os

import numpy as np
import pytest

from paper_2406_03726_b200 import errors as E
from paper_2406_03726_b200 import formats as F

CASES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "formats_cases.json")))


def _run(fn):
    try:
        return {"ok": fn()}
    except (E.ParseError, E.StructuralError) as e:
        return {"error": type(e).__name__, "line": getattr(e, "line_no", None)}


@pytest.mark.parametrize("case", CASES["edges"], ids=range(len(CASES["edges"])))
def test_parse_edge_list_matches_reference(case):
    def f():
        e = F.parse_edge_list(io.StringIO(case["text"]), F.ParseOptions(**case["opts"]), n_nodes=case["n_nodes"])
        return {"n_nodes": int(e.n_nodes), "rows": np.asarray(e.rows).tolist(), "cols": np.asarray(e.cols).tolist(),
                "weights": [float(x).hex() for x in np.asarray(e.weights)], "directed": bool(e.directed)}
    assert _run(f) == case["result"]


@pytest.mark.parametrize("case", CASES["labels"], ids=range(len(CASES["labels"])))
def test_parse_labels_matches_reference(case):
    def f():
        lv = F.parse_labels(io.StringIO(case["text"]), F.ParseOptions(**case["opts"]), k_classes=case["k_classes"],
                            n_nodes=case["n_nodes"])
        return {"labels": np.asarray(lv.labels).tolist(), "k_classes": int(lv.k_classes)}
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


def test_edge_list_and_labels_round_trip():
    rng = np.random.default_rng(4)
    n, m = 50, 300
    from paper_2406_03726_b200.graph import EdgeList, LabelVector
    e = EdgeList(n, rng.integers(0, n, m), rng.integers(0, n, m), rng.standard_normal(m) * 1e3, directed=True)
    buf = io.StringIO()
    F.write_edge_list(e, buf)
    back = F.parse_edge_list(io.StringIO(buf.getvalue()), F.ParseOptions(directed=True), n_nodes=n)
    assert np.array_equal(back.rows, e.rows) and np.array_equal(back.cols, e.cols)
    assert np.array_equal(back.weights, e.weights)
    lv = LabelVector(rng.integers(-1, 4, n), 4)
    buf = io.StringIO()
    F.write_labels(lv, buf)
    back = F.parse_labels(io.StringIO(buf.getvalue()), k_classes=4)
    assert np.array_equal(back.labels, lv.labels)


# ---- the bench / embed harness (bench_cli.py; cli.py:162-241) ----------------
def _files(tmp_path, edges, labels):
    e = tmp_path / "tri_edges.txt"
    lab = tmp_path / "tri_labels.txt"
    e.write_text(edges)
    lab.write_text(labels)
    return str(e), str(lab)


def test_cli_parse_error_exit_code(tmp_path, capsys):
    from paper_2406_03726_b200 import bench_cli
    e, lab = _files(tmp_path, "0 1\n0 x\n", "0\n1\n")
    assert bench_cli.main(["bench", "--edges", e, "--labels", lab]) == bench_cli.EXIT_PARSE
    assert "line 2" in capsys.readouterr().err
    e, lab = _files(tmp_path, "0 1\n1 2\n", "0\n1\n")  # 2 labels for 3 nodes
    assert bench_cli.main(["embed", "--edges", e, "--labels", lab, "--out", "-"]) == bench_cli.EXIT_SHAPE
    assert bench_cli.main(["bench", "--edges", e, "--labels", lab, "--repeats", "0"]) == bench_cli.EXIT_USAGE


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
    assert {x[1] for x in rows} == {"gpu", "gpu-ops"} and all(float(x[6]) > 0 for x in rows)
