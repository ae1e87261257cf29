"""GPU biclique-cover product (cmvg_bicover_matvec_f64, replacing the
reference's matvec_biclique_into, biclique.hpp:39-46) against the oracle
(oracle/pyoracle.py matvec_biclique) and matvec_csr: the spec's known answers,
random / planted / copy-model graphs, host and device pointers, and PageRank
on a cover of A^T against the oracle's CSR PageRank (the spec's kernel
agreement).  Tolerance: 1e-12 relative per entry (all terms
are positive, so the product is as accurate as matvec_csr)."""
import json
import os

import numpy as np
import pytest

import paper_1708_07271_b200 as P
from oracle import pyoracle as O
from tests.helpers import csr_from_rows, max_rel_err, oracle_csr, x_uniform

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.mark.parametrize("ex", GOLD["matvec_biclique"], ids=lambda e: e["spec"])
def test_spec_examples_on_gpu(cuda, ex):
    c = P.BicliqueCover.from_lists(ex["n"], ex["bicliques"], ex["residual"])
    y = c.matvec(np.asarray(ex["x"], dtype=np.float64))
    assert y.tolist() == ex["y"] and c.compressed_size == ex["adds"]


@pytest.mark.parametrize("per_round", [1, 0])
def test_copy_model_parity(cuda, per_round):
    import torch

    g = P.CsrGraph.copy_model(3000 if per_round else 1 << 15, 12.0, seed=9)
    c = P.BicliqueCover.extract_greedy(g, per_round=per_round)
    assert c.verify(g) and c.compressed_size < g.m
    x = x_uniform(g.n, 4)
    want = oracle_csr(g).matvec(x, 8)
    y = c.matvec(x)
    assert max_rel_err(y, want) <= 1e-12
    bl, res = c.lists()
    yo, _, adds = O.matvec_biclique(g.n, bl, res.tolist(), x) if g.n <= 4000 else (want, None, c.compressed_size)
    assert max_rel_err(y, yo) <= 1e-12 and adds == c.compressed_size
    yd = c.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(yd, y)  # host and device paths run the same kernels


def test_random_and_planted(cuda):
    rng = np.random.default_rng(1)
    for n, p in [(1, 0.0), (7, 0.5), (300, 0.05), (1024, 0.01)]:
        rows = [sorted(set(rng.choice(n, size=rng.binomial(n, p), replace=False).tolist())) for _ in range(n)]
        g = csr_from_rows(rows)
        c = P.BicliqueCover.extract_greedy(g, per_round=0)
        x = x_uniform(n, 2)
        assert max_rel_err(c.matvec(x), oracle_csr(g).matvec(x)) <= 1e-12
    rows = [set() for _ in range(2000)]
    S, T = rng.choice(2000, 300, replace=False), rng.choice(2000, 200, replace=False)
    for u in S:
        rows[u].update(T.tolist())
    g = csr_from_rows([sorted(r) for r in rows])
    c = P.BicliqueCover.extract_greedy(g)
    assert c.compressed_size <= 0.01 * g.m
    x = x_uniform(g.n, 3)
    assert max_rel_err(c.matvec(x), oracle_csr(g).matvec(x)) <= 1e-12


def test_dimension_error(cuda):
    c = P.BicliqueCover.from_lists(4, [([0, 1], [2, 3])], [])
    with pytest.raises(ValueError):
        c.matvec(np.zeros(3))


def test_pagerank_on_cover_of_transpose(cuda):
    """Power iteration with the biclique kernel on A^T agrees with the
    oracle's CSR PageRank (kernels agree within 1e-9)."""
    import torch

    g = P.CsrGraph.copy_model(4000, 10.0, seed=12)
    at = g.transpose()
    k = P.BicliqueKernel(P.BicliqueCover.extract_greedy(at, per_round=0))
    deg = g.out_degrees().astype(np.float64)
    n, alpha = g.n, 0.15
    p = torch.full((n,), 1.0 / n, dtype=torch.float64, device="cuda")
    d = torch.from_numpy(deg).cuda()
    y = torch.empty_like(p)
    for _ in range(30):
        q = torch.where(d > 0, p / torch.clamp(d, min=1.0), torch.zeros_like(p))
        k.multiply(q, y)
        dm = float(p[d == 0].sum())
        p = alpha / n + (1 - alpha) * (y + dm / n)
    want, _ = O.pagerank_csr(oracle_csr(at), g.out_degrees(), alpha, 30)
    assert np.max(np.abs(p.cpu().numpy() - want)) <= 1e-9
