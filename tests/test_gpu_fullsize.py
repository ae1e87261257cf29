"""GPU parity at the BASELINE.json sizes (configs[1..4]): every product of the
north star against the CPU oracle on the full graphs, in the driver's -m gpu
run.  Tolerances (BASELINE.json north_star): fp64 1e-12 relative per entry,
fp32 1e-5 relative per entry against fp64 matvec_csr (csr.hpp:48-55) of the
fp32-rounded x, empty rows exactly 0; PageRank 1e-12 per entry and
|sum p - 1| <= 1e-10 against pagerank(CsrKernel(A^T))
(pagerank.hpp:100-102).

  C2  n = 2^24, deg 20, R = 3: y = A x^T and y = x A in fp64 and fp32
  C3  n = 2^26, deg 24: 50 PageRank iterations on BV(A^T), alpha 0.15, kUniform
  C4  n = 2^25 social (power-law degrees, R = unbounded): y = A x^T in fp32
  C5  n = 2^27, deg 16: Y = A X with k = 16 (4 random columns checked)

Inputs are the seeded generators of SURVEY.md Appendix A (tests/helpers.py)."""
import numpy as np
import pytest

import paper_1708_07271_b200 as P
from oracle import pyoracle as O
from tests.helpers import CONFIGS, bv_params, make_graph, max_rel_err, x_uniform

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

F64_TOL = 1e-12
F32_TOL = 1e-5


def _oracle(g):
    return O.Csr.from_arrays(g.n, g.row_offsets, g.columns)


@pytest.fixture(scope="module")
def c2():
    g = make_graph(2)
    s = P.BvStream.encode(g, bv_params(2))
    return g, s, P.BvGraph(s)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_c2_gather_full_size(cuda, c2, dtype):
    import torch

    g, s, dg = c2
    assert g.n == CONFIGS[2]["n"]
    x = x_uniform(g.n, 21)
    if dtype == "f32":
        x = x.astype(np.float32)
    want = O.matvec_csr_raw(g.n, g.row_offsets, g.columns, x.astype(np.float64), O.threads())
    y = dg.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    assert max_rel_err(y, want) <= (F64_TOL if dtype == "f64" else F32_TOL)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_c2_scatter_full_size(cuda, c2, dtype):
    import torch

    g, s, dg = c2
    x = x_uniform(g.n, 22)
    if dtype == "f32":
        x = x.astype(np.float32)
    at = _oracle(g).transpose()
    want = at.matvec(x.astype(np.float64), O.threads())
    y = dg.matvec(torch.from_numpy(x).cuda(), form="scatter").cpu().numpy()
    assert max_rel_err(y, want) <= (F64_TOL if dtype == "f64" else F32_TOL)
    # the reference's way: (A^T) x on the transpose's compression (built on the GPU)
    y = dg.matvec(torch.from_numpy(x).cuda(), form="left").cpu().numpy()
    assert max_rel_err(y, want) <= (F64_TOL if dtype == "f64" else F32_TOL)


def test_c3_pagerank_full_size(cuda):
    g = make_graph(3)
    assert g.n == CONFIGS[3]["n"]
    at = g.transpose()
    dg = P.BvGraph(P.BvStream.encode(at, bv_params(3)))
    deg = g.out_degrees()
    p, it = dg.pagerank(deg, alpha=0.15, iterations=50)
    del dg
    want, _ = O.pagerank_csr(O.Csr.from_arrays(at.n, at.row_offsets, at.columns), deg.astype(np.uint32), 0.15, 50,
                             nthreads=O.threads())
    assert it == 50
    assert np.max(np.abs(p - want) / want) <= F64_TOL
    assert abs(p.sum() - 1.0) <= 1e-10


def test_c4_gather_f32_full_size(cuda):
    import torch

    g = make_graph(4)
    assert g.n == CONFIGS[4]["n"]
    s = P.BvStream.encode(g, bv_params(4))
    dg = P.BvGraph(s, P.CreateOptions(window=3968))  # a window the size of the 4096-row communities
    assert dg.info()["max_depth"] > 3  # unbounded reference chains (R = infinity)
    x = x_uniform(g.n, 23).astype(np.float32)
    want = O.matvec_csr_raw(g.n, g.row_offsets, g.columns, x.astype(np.float64), O.threads())
    y = dg.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    assert max_rel_err(y, want) <= F32_TOL


def test_c5_matmat_full_size(cuda):
    import torch

    g = make_graph(5)
    assert g.n == CONFIGS[5]["n"]
    dg = P.BvGraph(P.BvStream.encode(g, bv_params(5)))
    rng = np.random.default_rng(5)
    X = torch.rand((g.n, 16), dtype=torch.float32, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    Y = dg.matmat(X)
    for c in sorted(rng.choice(16, 4, replace=False).tolist()):
        xc = X[:, c].double().cpu().numpy()
        want = O.matvec_csr_raw(g.n, g.row_offsets, g.columns, xc, O.threads())
        assert max_rel_err(Y[:, c].double().cpu().numpy(), want) <= F32_TOL, c
