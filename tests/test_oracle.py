"""Pins the CPU oracle (the restated reference API) against every known answer
the reference ships for this path: the SPEC.md examples (tests/golden) and the
SPEC.md properties / acceptance criteria, at CPU-test sizes."""
import json
import os

import numpy as np
import pytest

from oracle import pyoracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def csr_of(rows):
    n = len(rows)
    ro = np.zeros(n + 1, dtype=np.uint64)
    ro[1:] = np.cumsum([len(r) for r in rows])
    cols = np.asarray([c for r in rows for c in r], dtype=np.uint32)
    return O.Csr.from_arrays(n, ro, cols)


def rows_of(g):
    return [g.row(u).tolist() for u in range(g.n)]


def rm_of(e):
    return O.RefMatrix.from_arrays(e["n"], e["refs"], e["plus"], e["minus"])


@pytest.mark.parametrize("e", GOLD["build_csr"], ids=lambda e: e["spec"])
def test_build_csr(e):
    g = O.Csr.build(e["edges"], e["n"])
    assert rows_of(g) == e["rows"]


def test_build_csr_out_of_range():
    with pytest.raises(IndexError, match="3"):
        O.Csr.build([(0, 1), (3, 0)], 3)


@pytest.mark.parametrize("e", GOLD["transpose"], ids=lambda e: e["spec"])
def test_transpose(e):
    assert rows_of(csr_of(e["rows"]).transpose()) == e["want"]


def test_transpose_involution():
    rng = np.random.default_rng(1)
    for _ in range(20):
        n = int(rng.integers(1, 64))
        edges = rng.integers(0, n, size=(int(rng.integers(0, 4 * n)), 2))
        g = O.Csr.build(edges, n)
        assert rows_of(g.transpose().transpose()) == rows_of(g)


@pytest.mark.parametrize("e", GOLD["out_degrees"], ids=lambda e: e["spec"])
def test_out_degrees(e):
    assert csr_of(e["rows"]).out_degrees().tolist() == e["want"]


@pytest.mark.parametrize("e", GOLD["matvec_csr"], ids=lambda e: e["spec"])
def test_matvec_csr(e):
    assert csr_of(e["rows"]).matvec(np.asarray(e["x"], float)).tolist() == e["y"]


def test_matvec_csr_dimension_error():  # csr.hpp:50
    with pytest.raises(ValueError):
        csr_of([[0]]).matvec(np.zeros(2))


def test_matvec_csr_partition_independent():
    g = O.Csr.build(np.random.default_rng(2).integers(0, 5000, size=(60000, 2)), 5000)
    x = np.random.default_rng(3).random(5000)
    assert np.array_equal(g.matvec(x, 1), g.matvec(x, 7))


@pytest.mark.parametrize("e", GOLD["compress"], ids=lambda e: e["spec"])
def test_compress(e):
    g = csr_of(e["rows"])
    rm = O.RefMatrix.compress(g, e["window"])
    refs, po, pc, mo, mc = rm.arrays()
    want_refs = [O.NO_REF if r is None else r for r in e["refs"]]
    assert refs.tolist() == want_refs
    assert [pc[po[i]:po[i + 1]].tolist() for i in range(g.n)] == e["plus"]
    assert [mc[mo[i]:mo[i + 1]].tolist() for i in range(g.n)] == e["minus"]
    assert len(pc) + len(mc) == e["m_prime"]
    rm.validate()


def test_compress_window_error():  # ref_matrix.hpp:67
    with pytest.raises(ValueError):
        O.RefMatrix.compress(csr_of([[0]]), 0)


@pytest.mark.parametrize("e", GOLD["reconstruct_row"], ids=lambda e: e["spec"])
def test_reconstruct_row(e):
    assert rm_of(e).reconstruct_row(e["row"]).tolist() == e["want"]


def test_reconstruct_row_out_of_range():  # ref_matrix.hpp:72
    e = GOLD["reconstruct_row"][0]
    with pytest.raises(IndexError):
        rm_of(e).reconstruct_row(e["n"])


@pytest.mark.parametrize("e", GOLD["stats"], ids=lambda e: e["spec"])
def test_stats(e):
    g = csr_of(e["rows"])
    s = O.RefMatrix.compress(g, e["window"]).stats(g)
    assert s["m"] == e["m"] and s["m_prime"] == e["m_prime"]
    assert s["ratio"] == pytest.approx(e["ratio"])
    assert s["ratio_by_convention"] == e["ratio_by_convention"]


@pytest.mark.parametrize("e", GOLD["matvec_ref"], ids=lambda e: e["spec"])
def test_matvec_ref(e):
    y, (adds, refs) = rm_of(e).matvec(np.asarray(e["x"], float))
    assert y.tolist() == e["y"]
    assert adds == e["adds"]


@pytest.mark.parametrize("e", GOLD["matvec_ref_left"], ids=lambda e: e["spec"])
def test_matvec_ref_left(e):
    g = csr_of(e["rows"])
    rm = O.RefMatrix.compress(g.transpose(), 7)
    y, _ = rm.matvec(np.asarray(e["x"], float))
    assert y.tolist() == e["y"]


def test_proposition1_random_corpus():  # SPEC.md:218,426-427 (acceptance 1-2, scaled to 200 graphs)
    rng = np.random.default_rng(11)
    for t in range(200):
        n = int(rng.integers(1, 200))
        dens = rng.uniform(0.01, 0.5)
        A = rng.random((n, n)) < dens
        u, v = np.nonzero(A)
        g = O.Csr.build(np.stack([u, v], 1), n)
        W = int(rng.integers(1, 33))
        rm = O.RefMatrix.compress(g, W)
        rm.validate()
        x = rng.uniform(-1, 1, n)
        y, (adds, refs) = rm.matvec(x)
        want = g.matvec(x)
        assert np.max(np.abs(y - want)) <= 1e-9 * (1 + np.max(np.abs(want), initial=0))
        st = rm.stats(g)
        assert adds == st["m_prime"] + refs  # SPEC.md:219 op-count law
        assert st["m_prime"] <= g.m
        back = rm.reconstruct_graph()
        assert np.array_equal(back.row_offsets, g.row_offsets) and np.array_equal(back.cols, g.cols)


def test_copy_chain_op_count():  # SPEC.md:428 (acceptance 3)
    n, base = 100_000, 100
    ro = np.arange(n + 1, dtype=np.uint64) * base
    cols = np.tile(np.arange(0, 2 * base, 2, dtype=np.uint32), n)
    g = O.Csr.from_arrays(n, ro, cols)
    rm = O.RefMatrix.compress(g, 1)
    st = rm.stats(g)
    assert st["m_prime"] == base
    _, (adds, refs) = rm.matvec(np.ones(n))
    assert adds == base + (n - 1) and refs == n - 1
    assert g.m / st["m_prime"] > 1e4  # the spec's "> 1e4" ratio is m/m' (m/adds is ~100)


def test_erdos_renyi_null():  # SPEC.md:430 (acceptance 5)
    rng = np.random.default_rng(5)
    n = 10_000
    g = O.Csr.build(rng.integers(0, n, size=(100_000, 2)), n)
    st = O.RefMatrix.compress(g, 7).stats(g)
    assert g.m / st["m_prime"] <= 1.2


def dense_pagerank(n, edges, alpha, iters, dangling="uniform"):
    A = np.zeros((n, n))
    for u, v in edges:
        A[u, v] = 1.0
    d = A.sum(1)
    p0 = np.full(n, 1 / n)
    p = p0.copy()
    for _ in range(iters):
        q = np.where(d > 0, p / np.where(d > 0, d, 1), 0)
        p = alpha * p0 + (1 - alpha) * (A.T @ q + (p[d == 0].sum() / n if dangling == "uniform" else 0))
    return p


@pytest.mark.parametrize("e", GOLD["pagerank"], ids=lambda e: e["spec"])
def test_pagerank_golden(e):
    g = O.Csr.build(e["edges"], e["n"])
    at, deg = g.transpose(), g.out_degrees()
    p, it = O.pagerank_csr(at, deg, e["alpha"], e["iterations"], dangling=e["dangling"])
    assert it == e["iterations"]
    assert np.max(np.abs(p - np.asarray(e["want"]))) <= e["tol"]
    p2, _ = O.pagerank_ref(O.RefMatrix.compress(at, 7), deg, e["alpha"], e["iterations"], dangling=e["dangling"])
    assert np.max(np.abs(p2 - np.asarray(e["want"]))) <= e["tol"]


def test_pagerank_dense_corpus():  # SPEC.md:431-432 (acceptance 6-7)
    rng = np.random.default_rng(9)
    for _ in range(40):
        n = int(rng.integers(1, 128))
        A = rng.random((n, n)) < rng.uniform(0.02, 0.3)
        u, v = np.nonzero(A)
        edges = np.stack([u, v], 1)
        g = O.Csr.build(edges, n)
        at, deg = g.transpose(), g.out_degrees()
        for pol in ("uniform", "drop"):
            want = dense_pagerank(n, edges, 0.15, 50, pol)
            p, _ = O.pagerank_csr(at, deg, 0.15, 50, dangling=pol)
            pr, _ = O.pagerank_ref(O.RefMatrix.compress(at, 5), deg, 0.15, 50, dangling=pol)
            assert np.max(np.abs(p - want)) <= 1e-10
            assert np.max(np.abs(pr - p)) <= 1e-9
            if pol == "uniform":
                assert abs(p.sum() - 1) <= 1e-10


def test_pagerank_errors():  # pagerank.hpp:96-98
    g = O.Csr.build([(0, 1)], 2)
    at, deg = g.transpose(), g.out_degrees()
    with pytest.raises(ValueError):
        O.pagerank_csr(at, deg, 1.0, 10)
    with pytest.raises(ValueError):
        O.pagerank_csr(at, deg, 0.15, 0)
    with pytest.raises(ValueError):
        O.pagerank_csr(at, deg, 0.15, 10, start=np.array([0.7, 0.7]))


def test_pagerank_l1_tolerance_stops_early():  # pagerank.hpp:94-95
    g = O.Csr.build([(0, 1), (1, 0)], 2)
    p, it = O.pagerank_csr(g.transpose(), g.out_degrees(), 0.15, 100, l1_tolerance=1e-6)
    assert it == 1 and np.allclose(p, 0.5)


def test_pagerank_uniform_fixpoint():
    n = 64
    edges = [(i, (i + 1) % n) for i in range(n)]
    g = O.Csr.build(edges, n)
    p, _ = O.pagerank_csr(g.transpose(), g.out_degrees(), 0.15, 30)
    assert np.max(np.abs(p - 1 / n)) <= 1e-12
