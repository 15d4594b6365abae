"""Command-line contract of the B200 engine (mirrors the reference's
pkg/tests/test_cli.py: flags, exact CSV/JSON schemas, exit codes, digest
invariance) and the edge-list ingest (graph_io.py:34-84).  Runs that touch
the device are marked gpu; usage errors and host-side generators run here."""

from __future__ import annotations

import json

import numpy as np
import pytest

from paper_1903_07754_b200.cli import CSV_HEADER, main


def run_cli(capsys, *argv):
    code = main(list(argv))
    cap = capsys.readouterr()
    return code, cap.out, cap.err


def csv_rows(out):
    lines = out.strip().splitlines()
    assert lines[0] == CSV_HEADER
    return lines[1:]


def digest_of(err):
    for line in err.splitlines():
        if line.startswith("# totals "):
            return json.loads(line[len("# totals "):])["digest"]
    raise AssertionError(err)


# ------------------------------------------------------------ CPU: usage ---
def test_usage_errors(capsys, tmp_path):
    assert run_cli(capsys, "run", "--app", "pagerank", "--gen", "path:4")[0] == 1
    code, _, err = run_cli(capsys, "run", "--app", "bfs", "--gen", "path:4")
    assert code == 1 and "root" in err
    assert run_cli(capsys, "run", "--app", "bfs", "--gen", "path:4", "--root", "9")[0] == 1
    code, _, err = run_cli(capsys, "run", "--app", "cc", "--graph", str(tmp_path / "missing.el"))
    assert code == 1 and "missing.el" in err
    f = tmp_path / "g.el"
    f.write_text("0 1\n")
    assert run_cli(capsys, "run", "--app", "cc", "--graph", str(f), "--gen", "path:4")[0] == 1
    assert run_cli(capsys, "sweep", "--app", "cc", "--gen", "grid:2:2", "--sweep", "threshold",
                   "--values", ",")[0] == 1
    assert run_cli(capsys, "generate", "--gen", "path:3", "--out", str(tmp_path / "no" / "dir" / "p.el"))[0] == 1
    assert run_cli(capsys, "run", "--app", "cc", "--gen", "bogus:1")[0] == 1


def test_generate_host_graphs(capsys, tmp_path):
    out = tmp_path / "p.el"
    assert run_cli(capsys, "generate", "--gen", "path:3", "--out", str(out))[0] == 0
    assert out.read_text() == "0 1\n1 2\n"
    g = tmp_path / "g.el"
    run_cli(capsys, "generate", "--gen", "grid:2:2", "--out", str(g))
    assert len(g.read_text().splitlines()) == 8


def test_parse_edge_list_semantics():
    import paper_1903_07754_b200 as wg
    el = wg.parse_edge_list("# vertices 6\n% comment\n0 1\n\n1 2\n# vertices 9\n")
    assert el.vertex_count == 6 and el.edge_count == 2 and not el.is_weighted()
    el = wg.parse_edge_list("0 3 5\n2 1 1\n")
    assert el.vertex_count == 4 and el.is_weighted() and list(el.edges()) == [(0, 3, 5), (2, 1, 1)]
    for bad, msg in (("0 1\n1 2 3\n", "line 2: mixed"), ("0\n", "line 1: expected"),
                     ("0 x\n", "non-integer"), ("-1 2\n", "negative"), ("0 1 0\n", "weight must be positive")):
        with pytest.raises(wg.ParseError, match=msg):
            wg.parse_edge_list(bad)
    # serialize is the inverse (header only when the count is not implied)
    for el in (wg.EdgeList(7, [0, 3], [1, 2]), wg.EdgeList(3, [0, 1], [1, 2], [4, 9])):
        back = wg.parse_edge_list(wg.serialize_edge_list(el))
        assert back.vertex_count == el.vertex_count and list(back.edges()) == list(el.edges())


def test_binary_edge_list_round_trip(tmp_path):
    import paper_1903_07754_b200 as wg
    el = wg.EdgeList(10, [0, 5, 9], [1, 2, 0], [3, 1, 7])
    p = tmp_path / "g.npz"
    wg.save_edge_list_binary(el, p)
    back = wg.load_edge_list(p)
    assert back.vertex_count == 10 and list(back.edges()) == list(el.edges())
    t = tmp_path / "g.el"
    t.write_text(wg.serialize_edge_list(el))
    assert list(wg.load_edge_list(t).edges()) == list(el.edges())


# ------------------------------------------------------------ GPU: runs ---
@pytest.mark.gpu
class TestRunGPU:
    def test_bfs_path8_rows_and_exit(self, capsys):
        code, out, _ = run_cli(capsys, "run", "--app", "bfs", "--gen", "path:8", "--root", "0")
        assert code == 0
        rows = csv_rows(out)
        assert len(rows) == 7
        for row in rows:
            f = row.split(",")
            assert len(f) == 7
            int(f[0]); float(f[2]); float(f[3]); float(f[4]); int(f[5]); int(f[6])

    def test_engines_agree_and_push_rejected(self, capsys):
        digests = set()
        for engine in ("wedge", "full"):
            code, _, err = run_cli(capsys, "run", "--app", "sssp", "--gen", "path:4", "--root", "0",
                                   "--engine", engine)
            assert code == 0
            digests.add(digest_of(err))
        assert len(digests) == 1
        code, _, err = run_cli(capsys, "run", "--app", "sssp", "--gen", "path:4", "--root", "0", "--engine", "push")
        assert code == 1 and "push" in err

    def test_max_iters_exit_code(self, capsys):
        code, out, _ = run_cli(capsys, "run", "--app", "bfs", "--gen", "path:16", "--root", "0", "--max-iters", "2")
        assert code == 2 and len(csv_rows(out)) == 2

    def test_json_format(self, capsys):
        code, out, _ = run_cli(capsys, "run", "--app", "cc", "--gen", "grid:3:3", "--format", "json")
        assert code == 0
        doc = json.loads(out)
        assert doc["totals"]["converged"] is True and doc["config"]["app"] == "cc"
        assert len(doc["iterations"]) == doc["totals"]["iterations"]

    def test_graph_file_and_binary(self, capsys, tmp_path):
        f = tmp_path / "g.el"
        f.write_text("0 1\n1 2\n2 3\n")
        code, out, err = run_cli(capsys, "run", "--app", "bfs", "--graph", str(f), "--root", "0")
        assert code == 0 and len(csv_rows(out)) == 3
        b = tmp_path / "g.npz"
        assert run_cli(capsys, "generate", "--gen", "path:4", "--out", str(b))[0] == 0
        code, out2, err2 = run_cli(capsys, "run", "--app", "bfs", "--graph", str(b), "--root", "0")
        assert code == 0 and digest_of(err2) == digest_of(err)

    def test_workers_env_default(self, capsys, monkeypatch):
        monkeypatch.setenv("WEDGE_WORKERS", "3")
        code, _, err = run_cli(capsys, "run", "--app", "cc", "--gen", "grid:2:2")
        cfg = json.loads([l for l in err.splitlines() if l.startswith("# config ")][0][len("# config "):])
        assert code == 0 and cfg["workers"] == 3

    def test_sweeps(self, capsys):
        code, out, _ = run_cli(capsys, "sweep", "--app", "cc", "--gen", "grid:16:16", "--sweep", "precision",
                               "--values", "1,2,4,8,16")
        rows = [r.split(",") for r in out.strip().splitlines()[1:]]
        assert code == 0 and len(rows) == 5 and len({r[-1] for r in rows}) == 1
        code, out, _ = run_cli(capsys, "sweep", "--app", "cc", "--gen", "grid:8:8", "--sweep", "threshold",
                               "--values", "0.0,1.0")
        _, z, o = out.strip().splitlines()
        z, o = z.split(","), o.split(",")
        assert code == 0 and int(z[2]) == 0
        assert int(o[2]) == int(o[1]) - 1 and int(o[3]) == 1 and z[-1] == o[-1]

    def test_generate_rmat_deterministic_and_weights(self, capsys, tmp_path):
        import paper_1903_07754_b200 as wg
        a, b = tmp_path / "a.el", tmp_path / "b.el"
        for f in (a, b):
            assert run_cli(capsys, "generate", "--gen", "rmat:4:8", "--seed", "1", "--out", str(f))[0] == 0
        assert a.read_text() == b.read_text()
        w = tmp_path / "w.el"
        assert run_cli(capsys, "generate", "--gen", "path:5", "--weights", "9", "--out", str(w))[0] == 0
        el = wg.parse_edge_list(w.read_text())
        assert el.is_weighted() and all(1 <= x <= 9 for *_, x in el.edges())

    def test_bench_runs(self, capsys):
        code, out, _ = run_cli(capsys, "bench", "--app", "bfs", "--gen", "rmat:8:8", "--root", "0")
        assert code == 0 and "b200" in out


@pytest.mark.gpu
@pytest.mark.parametrize("app,root", [("bfs", "0"), ("cc", None), ("sssp", "0")])
def test_digest_invariant_cross_product(capsys, app, root):
    """Engine, workers, threshold, precision and vector width never change results
    (reference test_cli.py:190-211, without the push engine)."""
    base = ["run", "--app", app, "--gen", "grid:4:4", "--format", "csv"] + (["--root", root] if root else [])
    digests = set()
    code, _, err = run_cli(capsys, *base, "--engine", "full")
    assert code == 0
    digests.add(digest_of(err))
    for threshold in ("0", "0.5", "1"):
        for precision in ("1", "8"):
            for width in ("1", "4"):
                code, _, err = run_cli(capsys, *base, "--engine", "wedge", "--threshold", threshold,
                                       "--precision", precision, "--vector-width", width, "--workers", "3")
                assert code == 0
                digests.add(digest_of(err))
    assert len(digests) == 1
