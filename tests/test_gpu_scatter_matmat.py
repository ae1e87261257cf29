"""GPU parity of the scatter form y = x A (on A's own compression; the
reference computes it as matvec_ref_left on compress(transpose(g)),
ref_matvec.hpp:37-41) and of the multi-vector product Y = A X (config 5,
k = 16, fp32) against the oracle's matvec_csr."""
import numpy as np
import pytest

import paper_1708_07271_b200 as P
from oracle import pyoracle as O
from tests.helpers import bv_params, csr_from_rows, make_graph, max_rel_err, oracle_csr, x_uniform

pytestmark = pytest.mark.gpu


def oracle_left(g, x):
    return oracle_csr(g).transpose().matvec(np.asarray(x, dtype=np.float64), 8)


@pytest.mark.parametrize("dtype,tol", [(np.float64, 1e-12), (np.float32, 1e-5)])
@pytest.mark.parametrize("cfg,n", [(2, 1 << 16), (1, (1 << 15) + 77), (4, 1 << 14)])
def test_scatter_matches_oracle(cuda, dtype, tol, cfg, n):
    g = make_graph(cfg, n=n)
    dg = P.BvGraph(P.BvStream.encode(g, bv_params(cfg)))
    x = x_uniform(g.n, 9).astype(dtype)
    y = dg.matvec(x, form="scatter")
    assert max_rel_err(y, oracle_left(g, x)) <= tol


def test_scatter_device_and_edge_cases(cuda):
    import torch

    for rows in ([[0]], [[], [], []], [list(range(0, 40, 3))] * 60 + [[]] * 5, [[1, 2, 3, 4, 5, 6], [0], []] + [[]] * 4):
        g = csr_from_rows(rows)
        dg = P.BvGraph(P.BvStream.encode(g, P.BvParams()))
        x = x_uniform(g.n, 2)
        assert max_rel_err(dg.matvec(x, form="scatter"), oracle_left(g, x)) <= 1e-12
    g = make_graph(2, n=1 << 15)
    dg = P.BvGraph(P.BvStream.encode(g, bv_params(2)), P.CreateOptions(window=256))  # many far columns
    x = x_uniform(g.n, 4)
    y = dg.matvec(torch.from_numpy(x).cuda(), form="scatter").cpu().numpy()
    assert max_rel_err(y, oracle_left(g, x)) <= 1e-12


@pytest.mark.parametrize("dtype,tol", [(np.float64, 1e-12), (np.float32, 1e-5)])
def test_scatter_heavy_and_split_targets_deterministic(cuda, dtype, tol):
    # a hub column hit by every row of a block (> 512 contributions: a
    # warp-wide heavy target), columns split over adjacent lanes, long rows
    # with far targets, intervals crossing the window edge; the result must be
    # bit-identical across runs (fixed-order segmented sums, no atomics)
    rng = np.random.default_rng(11)
    n = 5000

    def row(k):
        r = {7} | set(rng.integers(0, n, 3).tolist())
        if k % 97 == 0:
            r |= set(rng.integers(0, n, 700).tolist())
        if k % 13 == 0:
            a = int(rng.integers(0, n - 600))
            r |= set(range(a, a + 500))
        return sorted(r)
    g = csr_from_rows([row(k) for k in range(n)])
    x = x_uniform(g.n, 3).astype(dtype)
    for params in (P.BvParams(), P.BvParams(window=0)):  # window 0: no references, heavy targets
        s = P.BvStream.encode(g, params)
        dg = P.BvGraph(s)
        y1 = dg.matvec(x, form="scatter")
        y2 = dg.matvec(x, form="scatter")
        assert np.array_equal(y1.view(np.uint8), y2.view(np.uint8))
        assert max_rel_err(y1, oracle_left(g, x)) <= tol
    assert s.layout_info()["bvt_heavy_targets"] > 0


def test_scatter_shards_sum(cuda):
    g = make_graph(2, n=(1 << 15) + 10)
    s = P.BvStream.encode(g, bv_params(2))
    x = x_uniform(g.n, 6)
    tot = np.zeros(g.n)
    for a, b in ((0, 16384), (16384, g.n)):
        tot += P.BvGraph(s, P.CreateOptions(row_begin=a, row_end=b)).matvec(x, form="scatter")
    assert max_rel_err(tot, oracle_left(g, x)) <= 1e-12


@pytest.mark.parametrize("k", [16, 4, 1, 32])
def test_matmat_matches_oracle(cuda, k):
    g = make_graph(5, n=1 << 15)
    dg = P.BvGraph(P.BvStream.encode(g, bv_params(5)))
    rng = np.random.default_rng(k)
    X = rng.random((g.n, k), dtype=np.float32)
    Y = dg.matmat(X)
    og = oracle_csr(g)
    for c in range(k):
        want = og.matvec(X[:, c].astype(np.float64), 8)
        assert max_rel_err(Y[:, c], want) <= 1e-5, c


def test_matmat_device_and_social(cuda):
    import torch

    g = make_graph(4, n=1 << 14)  # unbounded chains
    dg = P.BvGraph(P.BvStream.encode(g, bv_params(4)))
    X = np.random.default_rng(1).random((g.n, 16), dtype=np.float32)
    Y = dg.matmat(torch.from_numpy(X).cuda()).cpu().numpy()
    og = oracle_csr(g)
    for c in (0, 7, 15):
        assert max_rel_err(Y[:, c], og.matvec(X[:, c].astype(np.float64), 8)) <= 1e-5


@pytest.mark.parametrize("params", [dict(window=1, max_ref=1, min_interval=2, segment_rows=256),
                                    dict(window=3, max_ref=0, min_interval=3, segment_rows=512),
                                    dict(window=7, max_ref=2, min_interval=6, segment_rows=1024),
                                    dict(window=0, max_ref=3, min_interval=4, segment_rows=1024)])
def test_products_across_bv_params(cuda, params):
    # every product on streams encoded with other BV parameters (window w,
    # chain bound R, minimum interval Lmin, segment length)
    g = make_graph(2, n=(1 << 15) + 123)
    s = P.BvStream.encode(g, P.BvParams(**params))
    dg = P.BvGraph(s)
    x = x_uniform(g.n, 17)
    assert max_rel_err(dg.matvec(x), oracle_csr(g).matvec(x, 8)) <= 1e-12
    assert max_rel_err(dg.matvec(x, form="scatter"), oracle_left(g, x)) <= 1e-12
    X = np.stack([x_uniform(g.n, 30 + c) for c in range(3)], 1).astype(np.float32)
    Y = dg.matmat(X)
    for c in range(3):
        assert max_rel_err(Y[:, c], oracle_csr(g).matvec(X[:, c].astype(np.float64), 8)) <= 1e-5
    ro, co = dg.decode_csr()
    assert np.array_equal(ro, g.row_offsets) and np.array_equal(co, g.columns)
