"""The CLI's GPU subcommands: matvec against the oracle,
pagerank with each kernel (csr / ref / biclique) agreeing, and the Table-1
bench TSV (ratio and S recomputable from the columns)."""
import numpy as np
import pytest

import paper_1708_07271_b200 as P
from oracle import pyoracle as O
from paper_1708_07271_b200 import cli

pytestmark = pytest.mark.gpu


def test_cli_matvec_matches_oracle(cuda, tmp_path, capsys):
    txt, cbv, yf = str(tmp_path / "g.txt"), str(tmp_path / "g.cbv"), str(tmp_path / "y.txt")
    assert cli.main(["gen", "--n", "5000", "--degree", "12", "--out", txt]) == 0
    assert cli.main(["compress", "--out", cbv, txt]) == 0
    for form in ("gather", "scatter"):
        assert cli.main(["matvec", "--uniform", "--seed", "3", "--form", form, "--out", yf, cbv]) == 0
        y = np.loadtxt(yf)
        g = cli.load_edge_list(txt)
        x = cli._vector(type("A", (), {"vector": None, "seed": 3})(), g.n)
        gg = g if form == "gather" else g.transpose()
        want = O.matvec_csr_raw(gg.n, gg.row_offsets, gg.columns, x, 1)
        assert np.max(np.abs(y - want) / np.maximum(np.abs(want), 1e-300)) <= 1e-12


def test_cli_pagerank_kernels_agree(cuda, tmp_path, capsys):
    txt = str(tmp_path / "g.txt")
    assert cli.main(["gen", "--n", "3000", "--degree", "8", "--out", txt]) == 0
    ranks = {}
    for k in ("ref", "csr", "biclique"):
        out = str(tmp_path / f"p_{k}.txt")
        assert cli.main(["pagerank", "--kernel", k, "--iters", "30", "--out", out, txt]) == 0
        ranks[k] = np.loadtxt(out)
    assert abs(ranks["ref"].sum() - 1.0) < 1e-10
    assert np.max(np.abs(ranks["ref"] - ranks["csr"])) < 1e-12
    assert np.max(np.abs(ranks["ref"] - ranks["biclique"])) < 1e-12


def test_cli_bench_tsv(cuda, tmp_path, capsys):
    txt = str(tmp_path / "g.txt")
    assert cli.main(["gen", "--n", "4000", "--degree", "10", "--out", txt]) == 0
    capsys.readouterr()
    assert cli.main(["bench", "--reps", "2", "--iters", "10", txt]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == cli.BENCH_HEADER
    f = dict(zip(lines[0].split("\t"), lines[1].split("\t")))
    assert int(f["m"]) > 0 and abs(float(f["ratio"]) - int(f["m"]) / int(f["m_prime"])) < 1e-3
    assert abs(float(f["S"]) - float(f["t"]) / float(f["t_prime"])) < 1e-2 * float(f["S"])
    assert float(f["linf"]) < 1e-12
