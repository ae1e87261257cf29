"""Biclique covers (reference include/cmv/biclique.hpp,
SPEC.md:296-357) on the CPU: the oracle's matvec_biclique / verify_cover
against the spec's known answers (tests/golden/spec_examples.json), the
product-side extraction, verification and BCV1 container against the oracle
and the spec's properties (exact coverage over random graphs, compressed_size
<= m, the planted K_{50,50} bound, kernel equivalence with matvec_csr).  The
GPU product is in test_gpu_biclique.py."""
import json
import os

import numpy as np
import pytest

import paper_1708_07271_b200 as P
from oracle import pyoracle as O
from tests.helpers import csr_from_rows, oracle_csr

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def rows_of(n, edges):
    rows = [[] for _ in range(n)]
    for u, v in sorted(set(map(tuple, edges))):
        rows[u].append(v)
    return rows


def cover_rows(g):
    ro, co = g.row_offsets, g.columns
    return [list(co[ro[u]:ro[u + 1]]) for u in range(g.n)]


def random_graph(rng, n, p):
    rows = [sorted(set(rng.choice(n, size=rng.binomial(n, p), replace=False).tolist())) for _ in range(n)]
    return csr_from_rows(rows)


def planted(rng, n, s, t, noise):
    rows = [set() for _ in range(n)]
    S = rng.choice(n, size=s, replace=False)
    C = rng.choice(n, size=t, replace=False)
    for u in S:
        rows[u].update(C.tolist())
    for _ in range(noise):
        rows[rng.integers(n)].add(int(rng.integers(n)))
    return csr_from_rows([sorted(r) for r in rows])


@pytest.mark.parametrize("ex", GOLD["matvec_biclique"], ids=lambda e: e["spec"])
def test_oracle_matvec_biclique_spec(ex):
    y, c, adds = O.matvec_biclique(ex["n"], ex["bicliques"], ex["residual"], ex["x"])
    assert y.tolist() == ex["y"] and c == ex["c"] and adds == ex["adds"]
    assert adds <= ex["m"]


@pytest.mark.parametrize("ex", GOLD["verify_cover"], ids=lambda e: e["spec"])
def test_verify_cover_spec(ex):
    rows = rows_of(ex["n"], ex["edges"])
    assert O.verify_cover(ex["n"], ex["bicliques"], ex["residual"], rows) == ex["want"]
    g = csr_from_rows(rows)
    try:
        c = P.BicliqueCover.from_lists(ex["n"], ex["bicliques"], ex["residual"])
    except ValueError:
        assert not ex["want"]
        return
    assert c.verify(g) == ex["want"]


def test_extract_k33_single_biclique():
    ex = GOLD["extract_greedy"][0]
    g = csr_from_rows(rows_of(ex["n"], ex["edges"]))
    c = P.BicliqueCover.extract_greedy(g)
    bl, res = c.lists()
    assert [(s.tolist(), t.tolist()) for s, t in bl] == [tuple(b) for b in ex["bicliques"]]
    assert len(res) == 0 and c.compressed_size == ex["compressed_size"] and g.m == ex["m"]
    assert c.verify(g)


def test_extract_overlapping_bicliques_disjoint():
    ex = GOLD["extract_greedy"][1]
    g = csr_from_rows(rows_of(ex["n"], ex["edges"]))
    for per_round in (1, 0):
        c = P.BicliqueCover.extract_greedy(g, per_round=per_round)
        bl, res = c.lists()
        assert c.verify(g) is True
        assert O.verify_cover(g.n, bl, res.tolist(), cover_rows(g))
        assert c.compressed_size <= g.m


def test_extract_nothing_to_share():
    g = csr_from_rows([[1], [2], [3], [0]])  # a cycle: no shared neighbourhoods
    c = P.BicliqueCover.extract_greedy(g)
    bl, res = c.lists()
    assert bl == [] and res.tolist() == [[0, 1], [1, 2], [2, 3], [3, 0]] and c.verify(g)


def test_extract_random_graphs_property():
    """Exact coverage and size sanity on random graphs."""
    rng = np.random.default_rng(7)
    for k in range(120):
        n = int(rng.integers(2, 80))
        g = random_graph(rng, n, float(rng.uniform(0.02, 0.5)))
        c = P.BicliqueCover.extract_greedy(g, per_round=int(k % 2))
        bl, res = c.lists()
        assert c.verify(g), k
        assert O.verify_cover(g.n, bl, res.tolist(), cover_rows(g)), k
        assert c.compressed_size <= g.m
        for s, t in bl:
            assert len(s) * len(t) > len(s) + len(t)


def test_extract_planted_biclique_bound():
    """K_{50,50} plus noise: compressed_size <= 0.1 m."""
    rng = np.random.default_rng(3)
    g = planted(rng, 400, 50, 50, 150)
    c = P.BicliqueCover.extract_greedy(g)
    assert c.verify(g)
    assert c.compressed_size <= 0.1 * g.m, (c.compressed_size, g.m)


def test_min_gain_and_max_rounds():
    rng = np.random.default_rng(5)
    g = planted(rng, 200, 20, 20, 50)
    c0 = P.BicliqueCover.extract_greedy(g, max_rounds=0)
    assert c0.lists()[0] == [] and c0.compressed_size == g.m and c0.verify(g)
    big = P.BicliqueCover.extract_greedy(g, min_gain=10 ** 9)
    assert big.lists()[0] == []
    with pytest.raises(ValueError):
        P.BicliqueCover.extract_greedy(g, min_gain=0)


def test_oracle_kernel_equivalence_random():
    """matvec_biclique = matvec_csr within 1e-9 relative-inf."""
    rng = np.random.default_rng(11)
    for _ in range(20):
        n = int(rng.integers(2, 200))
        g = random_graph(rng, n, 0.2)
        c = P.BicliqueCover.extract_greedy(g, per_round=0)
        bl, res = c.lists()
        x = rng.random(n)
        y, _, adds = O.matvec_biclique(n, bl, res.tolist(), x)
        want = oracle_csr(g).matvec(x)
        assert np.max(np.abs(y - want)) <= 1e-9 * max(1.0, np.max(np.abs(want)))
        assert adds == c.compressed_size


def test_bcv1_roundtrip_and_errors(tmp_path):
    rng = np.random.default_rng(2)
    g = planted(rng, 120, 12, 9, 60)
    c = P.BicliqueCover.extract_greedy(g)
    p = tmp_path / "c.bcv"
    c.save(str(p))
    text = p.read_text()
    assert text.startswith(f"BCV1 {g.n}\n") and "\nR\n" in text
    d = P.BicliqueCover.load(str(p))
    bl, res = c.lists()
    bl2, res2 = d.lists()
    assert [(a.tolist(), b.tolist()) for a, b in bl] == [(a.tolist(), b.tolist()) for a, b in bl2]
    assert np.array_equal(res, res2) and d.verify(g)
    d.save(str(tmp_path / "d.bcv"))
    assert (tmp_path / "d.bcv").read_text() == text  # deterministic serialisation
    bad = tmp_path / "bad.bcv"
    bad.write_text("XCV1 3\nR\n")
    with pytest.raises(P.FormatError):
        P.BicliqueCover.load(str(bad))
    for body in ["BCV1 3\nB 1\n0\n", "BCV1 3\nB 1\n0\n2 1\nR\n", "BCV1 3\nR\n0 5\n", "BCV1 3\nR\n1 0\n0 1\n",
                 "BCV1 3\nB 2\n1 0\n1 2\nR\n", "BCV1 3\n"]:
        bad.write_text(body)
        with pytest.raises(P.CorruptionError):
            P.BicliqueCover.load(str(bad))


def test_from_lists_validation():
    with pytest.raises(ValueError):
        P.BicliqueCover.from_lists(4, [([1, 0], [2])], [])  # sources not ascending
    with pytest.raises(IndexError):
        P.BicliqueCover.from_lists(4, [([0], [9])], [])  # out of range
    with pytest.raises(ValueError):
        P.BicliqueCover.from_lists(4, [([], [2])], [])  # empty side
