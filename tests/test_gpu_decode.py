"""GPU BV decode (bv_decode_csr) is bit-exact against the source adjacency
(the counterpart of reconstruct_graph, ref_matrix.hpp:75-76)."""
import numpy as np
import pytest

import paper_1708_07271_b200 as P
from tests.helpers import bv_params, csr_from_rows, make_graph

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,n", [(1, 1 << 16), (2, (1 << 16) + 5), (4, 1 << 15)])
def test_decode_bit_exact(cuda, cfg, n):
    g = make_graph(cfg, n=n)
    s = P.BvStream.encode(g, bv_params(cfg))
    dg = P.BvGraph(s)
    ro, co = dg.decode_csr()
    assert np.array_equal(ro, g.row_offsets)
    assert np.array_equal(co, g.columns)


def test_decode_device_buffers(cuda):
    import torch

    g = make_graph(1, n=1 << 15)
    dg = P.BvGraph(P.BvStream.encode(g, bv_params(1)))
    ro = torch.empty(g.n + 1, dtype=torch.int64, device="cuda")
    co = torch.empty(g.m, dtype=torch.int32, device="cuda")
    dg.decode_csr_device(ro, co)
    torch.cuda.synchronize()
    assert np.array_equal(ro.cpu().numpy().view(np.uint64), g.row_offsets)
    assert np.array_equal(co.cpu().numpy().view(np.uint32), g.columns)


def test_decode_edge_cases(cuda):
    for rows in ([[]], [[0]], [[], [1], [0, 1]], [list(range(40))] * 50 + [[]] * 3):
        g = csr_from_rows(rows)
        for params in (P.BvParams(), P.BvParams(max_ref=0), P.BvParams(window=1, segment_rows=2)):
            dg = P.BvGraph(P.BvStream.encode(g, params), P.CreateOptions(block_rows=1024))
            ro, co = dg.decode_csr()
            assert np.array_equal(ro, g.row_offsets) and np.array_equal(co, g.columns)


def test_decode_rejects_corruption(cuda):
    g = make_graph(1, n=1 << 12)
    s = P.BvStream.encode(g, bv_params(1))
    w = s.words()
    w[len(w) // 2] ^= 0xFFFF0000  # flip bits mid-stream
    bad = P.BvStream.from_words(g.n, g.m, s.params, w, s.stats()["stream_bits"], s.segment_offsets())
    with pytest.raises((P.CorruptionError, ValueError, IndexError)):
        P.BvGraph(bad)  # the host builder validates the stream first


def test_decode_long_rows_and_lists(cuda):
    """Rows with > 512 residuals, > 1024 copied entries, > 64 intervals and
    > 128 copy blocks next to short rows; bit-exact."""
    rng = np.random.default_rng(21)
    n = 6000
    rows = [sorted(set(rng.integers(0, n, 5).tolist())) for _ in range(n)]
    big = sorted(set(rng.integers(0, n, 2600).tolist()))
    rows[100] = big                                     # > 512 residuals
    rows[101] = big[:-3]                                # copies > 1024 entries of row 100
    rows[102] = big[::2]                                # many alternating copy blocks vs row 100
    rows[2000] = sorted(set(x for a in range(0, 5000, 60) for x in range(a, a + 5)))  # > 64 intervals
    rows[2001] = rows[2000][:-40] + [5990]
    g = csr_from_rows(rows)
    s = P.BvStream.encode(g, P.BvParams())
    ro, co = P.BvGraph(s).decode_csr()
    assert np.array_equal(ro, g.row_offsets) and np.array_equal(co, g.columns)


@pytest.mark.parametrize("cap", ["0", "4096"])
def test_decode_unstaged_tiles(cuda, monkeypatch, cap):
    """Tiles whose edges exceed the shared-memory staging buffer decode straight
    into the output columns (CMVG_DECODE_CAP shrinks the buffer); bit-exact."""
    monkeypatch.setenv("CMVG_DECODE_CAP", cap)
    for cfg, n in ((2, (1 << 15) + 3), (4, 1 << 14)):
        g = make_graph(cfg, n=n)
        ro, co = P.BvGraph(P.BvStream.encode(g, bv_params(cfg))).decode_csr()
        assert np.array_equal(ro, g.row_offsets) and np.array_equal(co, g.columns)


def test_decode_serial_matches(cuda, monkeypatch):
    """The serial thread-per-segment decoder (CMVG_SERIAL_DECODE) gives the same CSR."""
    monkeypatch.setenv("CMVG_SERIAL_DECODE", "1")
    g = make_graph(1, n=1 << 14)
    ro, co = P.BvGraph(P.BvStream.encode(g, bv_params(1))).decode_csr()
    assert np.array_equal(ro, g.row_offsets) and np.array_equal(co, g.columns)
