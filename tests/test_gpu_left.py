"""x A the reference's way (matvec_ref_left, ref_matvec.hpp:37-41: (A^T) x on
compress(transpose(g))) with everything on the GPU: A decoded from its BV
stream, transposed by a stable sort, references for A^T chosen by
cmv::compress's rule (ref_matrix.hpp:58-69) and its BV-F layout built by the
device builder; then the gather kernel.  Parity against the oracle's
matvec_csr(transpose(g)) (csr.hpp:48-55), fp64 <= 1e-12 and fp32 <= 1e-5 per
entry, empty columns exactly 0, repeated calls bit-identical."""
import numpy as np
import pytest

import paper_1708_07271_b200 as P
from tests.helpers import bv_params, csr_from_rows, make_graph, max_rel_err, oracle_csr, x_uniform

pytestmark = pytest.mark.gpu


def oracle_left(g, x):
    return oracle_csr(g).transpose().matvec(np.asarray(x, dtype=np.float64), 8)


@pytest.mark.parametrize("dtype,tol", [(np.float64, 1e-12), (np.float32, 1e-5)])
@pytest.mark.parametrize("cfg,n", [(2, 1 << 16), (1, (1 << 15) + 77), (3, 1 << 15), (4, 1 << 14), (5, 1 << 15)])
def test_left_matches_oracle(cuda, dtype, tol, cfg, n):
    g = make_graph(cfg, n=n)
    dg = P.BvGraph(P.BvStream.encode(g, bv_params(cfg)))
    x = x_uniform(g.n, 9).astype(dtype)
    want = oracle_left(g, x)
    y = dg.matvec(x, form="left")
    assert max_rel_err(y, want) <= tol
    assert np.all(y[want == 0] == 0)
    assert np.array_equal(dg.matvec(x, form="left"), y)  # deterministic


def test_left_device_pointers_and_edge_cases(cuda):
    import torch

    for rows in ([[0]], [[], [], []], [list(range(0, 40, 3))] * 60 + [[]] * 5, [[1, 2, 3, 4, 5, 6], [0], []] + [[]] * 4):
        g = csr_from_rows(rows)
        dg = P.BvGraph(P.BvStream.encode(g, P.BvParams()))
        x = x_uniform(g.n, 2)
        assert max_rel_err(dg.matvec(x, form="left"), oracle_left(g, x)) <= 1e-12
    rng = np.random.default_rng(3)
    n = 4000
    rows = [sorted(set(rng.integers(max(0, i - 50), min(n, i + 50), 10).tolist())) for i in range(n)]
    rows[7] = list(range(n))  # column hub of A^T everywhere: every row of A^T holds 7
    g = csr_from_rows(rows)
    for window in (1536, 256):
        dg = P.BvGraph(P.BvStream.encode(g, P.BvParams()), P.CreateOptions(window=window))
        x = x_uniform(g.n, 4)
        y = dg.matvec(torch.from_numpy(x).cuda(), form="left").cpu().numpy()
        assert max_rel_err(y, oracle_left(g, x)) <= 1e-12


def test_left_needs_whole_graph(cuda):
    g = make_graph(2, n=1 << 13)
    dg = P.BvGraph(P.BvStream.encode(g, bv_params(2)), P.CreateOptions(row_begin=0, row_end=4096))
    with pytest.raises(ValueError):
        dg.matvec(x_uniform(g.n, 1), form="left")
