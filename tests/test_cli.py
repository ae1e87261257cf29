"""CLI and edge-list ingestion (the reference's cli-io module):
load_edge_list / build_csr known answers and errors, and the host-side
subcommands (gen, compress, stats); the GPU subcommands run under -m gpu."""
import os

import numpy as np
import pytest

import paper_1708_07271_b200 as P
from paper_1708_07271_b200 import cli


def _write(tmp_path, text, name="g.txt"):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def _rows(g):
    ro, co = g.row_offsets, g.columns
    return [co[ro[i]:ro[i + 1]].tolist() for i in range(g.n)]


def test_build_csr_spec_examples():
    # SPEC.md:52-54
    assert _rows(cli.build_csr(np.zeros((0, 2)), 3)) == [[], [], []]
    assert _rows(cli.build_csr([(0, 1), (0, 1), (1, 0)], 2)) == [[1], [0]]
    assert _rows(cli.build_csr([(0, 2), (0, 1), (1, 2)], 3)) == [[1, 2], [2], []]
    with pytest.raises(IndexError):
        cli.build_csr([(0, 3)], 3)


def test_load_edge_list_examples_and_errors(tmp_path):
    g = cli.load_edge_list(_write(tmp_path, "0 1\n1 0\n"))  # 2-cycle
    assert g.n == 2 and _rows(g) == [[1], [0]]
    g = cli.load_edge_list(_write(tmp_path, "# comment\n0 2\n"))  # n = 3, one edge
    assert g.n == 3 and g.m == 1
    g = cli.load_edge_list(_write(tmp_path, "0 1  # trailing comment\n\n3 3\n"), n=6)
    assert g.n == 6 and _rows(g) == [[1], [], [], [3], [], []]
    with pytest.raises(cli.EdgeListError, match="line 2"):
        cli.load_edge_list(_write(tmp_path, "0 1\n0 x\n"))
    with pytest.raises(cli.EdgeListError, match="line 1"):
        cli.load_edge_list(_write(tmp_path, "0 1 2\n"))
    with pytest.raises(IndexError):
        cli.load_edge_list(_write(tmp_path, "0 5\n"), n=3)


def test_edge_list_round_trip(tmp_path):
    g = P.CsrGraph.copy_model(3000, 8.0, seed=5)
    path = str(tmp_path / "g.txt")
    cli.save_edge_list(g, path)
    h = cli.load_edge_list(path, n=g.n)
    assert np.array_equal(h.row_offsets, g.row_offsets) and np.array_equal(h.columns, g.columns)


def test_cli_gen_compress_stats(tmp_path, capsys):
    txt, cbv = str(tmp_path / "g.txt"), str(tmp_path / "g.cbv")
    assert cli.main(["gen", "--model", "copy", "--n", "2000", "--degree", "10", "--out", txt]) == 0
    assert cli.main(["compress", "--window", "7", "--out", cbv, txt]) == 0
    assert os.path.getsize(cbv) > 0
    capsys.readouterr()
    assert cli.main(["stats", cbv]) == 0
    out = capsys.readouterr().out.splitlines()
    assert out[0].split("\t")[:4] == ["n", "m", "m_prime", "ratio"]
    n, m, mp = (int(v) for v in out[1].split("\t")[:3])
    g = cli.load_edge_list(txt)
    assert (n, m) == (g.n, g.m) and mp > 0
    s = P.BvStream.load(cbv).decode_host()
    assert np.array_equal(s.columns, g.columns)


def test_cli_gen_er_and_errors(tmp_path, capsys):
    txt = str(tmp_path / "er.txt")
    assert cli.main(["gen", "--model", "er", "--n", "500", "--degree", "4", "--out", txt]) == 0
    g = cli.load_edge_list(txt, n=500)
    assert 1000 < g.m < 3000  # ~ n * degree
    assert cli.main(["stats", str(tmp_path / "missing.txt")]) == 1
    assert "error" in capsys.readouterr().err
    bad = _write(tmp_path, "0 1\nfoo\n", "bad.txt")
    assert cli.main(["compress", "--out", str(tmp_path / "b.cbv"), bad]) == 1
