"""BV-F (flat term stream of the gather / PageRank kernels, host/layout.hpp):
the layout built on the host, re-evaluated on the CPU with the kernel's exact
arithmetic (tests/layout_ref.py gather_bvf), must give A x within the fp64
tolerance (1e-12 relative, empty rows exactly 0) against the oracle's
matvec_csr (reference csr.hpp:48-55), and its structure must hold: one row end
per row, chunk start rows, escape segments."""
import numpy as np
import pytest

import paper_1708_07271_b200 as P
from tests.helpers import bv_params, csr_from_rows, make_graph, max_rel_err, oracle_csr, x_uniform
from tests.layout_ref import BVF_END, bvf_block, gather_bvf


def _check(g, params, window=1536, x=None, B=1024, max_depth=3):
    s = P.BvStream.encode(g, params)
    words, blocks = s.layout_export(P.CreateOptions(block_rows=B, window=window), kind="bvf")
    x = x_uniform(g.n, 3) if x is None else x
    y = gather_bvf(words, blocks, g.n, B, window, x, max_depth=max_depth)
    want = oracle_csr(g).matvec(x)
    assert max_rel_err(y, want) <= 1e-12
    # structure: one end per row, chunk start rows consistent with the ends
    for b in range(len(blocks)):
        info, sr, r, slots, escstart, esccol, chunks = bvf_block(words, blocks[b])
        nr = min(B, g.n - b * B)
        ends = [int(np.sum((c & BVF_END) != 0)) for c in chunks]
        # rows have an even number of terms: a row ends only on a word's high term
        assert all(not np.any(c[0::2] & BVF_END) for c in chunks)
        assert sum(ends) == nr
        assert info["nact"] <= 256 and info["K"] % 16 == 0
        row = 0
        for t in range(info["nact"]):
            assert int(sr[t]) == row
            row += ends[t]
    return s, words, blocks


@pytest.mark.parametrize("cfg,n", [(1, 6000), (2, 9000), (3, 7000), (5, 5000)])
def test_bvf_copy_model_matches_oracle(cfg, n):
    _check(make_graph(cfg, n=n), bv_params(cfg))


def test_bvf_social_unbounded_chains_and_escapes():
    g = make_graph(4, n=12000)
    s, words, blocks = _check(g, bv_params(4), max_depth=1 << 30)
    info = s.layout_info()
    assert info["max_depth"] > 3


@pytest.mark.parametrize("window", [3072, 3968])
def test_bvf_wide_window_social(window):
    # community-sized windows (the power-law C4 graph's 4096-row communities)
    g = make_graph(4, n=9000)
    _check(g, bv_params(4), window=window, max_depth=1 << 30)


def test_bvf_small_window_forces_slots_and_escapes():
    # a narrow window puts most columns outside it: far slots, then escapes
    g = make_graph(2, n=6000)
    s, words, blocks = _check(g, bv_params(2), window=256)
    flags = [bvf_block(words, blocks[b])[0]["flags"] for b in range(len(blocks))]
    assert any(f & 1 for f in flags)


def test_bvf_edge_rows_hub_and_empty():
    rng = np.random.default_rng(5)
    n = 3000
    rows = []
    for i in range(n):
        if i % 97 == 0:
            rows.append([])
        elif i == 1500:
            rows.append(sorted(set(rng.integers(0, n, 2500).tolist())))  # hub spanning many chunks
        elif i % 5 == 1 and i > 1:
            rows.append(list(rows[i - 1]))  # exact copy of the previous row: empty differential
        else:
            base = max(0, i - 40)
            rows.append(sorted(set(rng.integers(base, min(n, base + 90), 12).tolist())))
    g = csr_from_rows(rows)
    _check(g, P.BvParams())


def test_bvf_signed_values_and_cancellation():
    g = make_graph(2, n=5000)
    rng = np.random.default_rng(9)
    # signed entries over ~2^29 of dynamic range inside every window: the split
    # sums are exact here (the error left scales with G = 2^(E - cbits) times
    # the window's prefix rounding)
    x = rng.standard_normal(g.n) * np.exp(rng.uniform(-10, 10, g.n))
    s = P.BvStream.encode(g, bv_params(2))
    words, blocks = s.layout_export(P.CreateOptions(), kind="bvf")
    y = gather_bvf(words, blocks, g.n, 1024, 1536, x)
    want = oracle_csr(g).matvec(x)
    # signed sums of wide range: compare against the exact sum (fsum) per row
    import math
    ro, co = g.row_offsets, g.columns
    exact = np.array([math.fsum(x[co[ro[i]:ro[i + 1]]]) for i in range(g.n)])
    scale = np.array([np.sum(np.abs(x[co[ro[i]:ro[i + 1]]])) for i in range(g.n)])
    assert np.all(np.abs(y - exact) <= 1e-15 * scale + 1e-300)
    assert np.all(np.abs(want - exact) <= 1e-13 * scale + 1e-300)


@pytest.mark.parametrize("window,lmin", [(16, 2), (16, 4), (64, 2), (1536, 2)])
def test_bvf_builder_bounds_adversarial(window, lmin):
    """The shared block builder (host/bvf_block.hpp) runs in arenas sized by
    its worst-case bounds (the device build allocates exactly those): windows
    of 16 columns (nearly every column far: slots, then escapes), intervals as
    short as the encoder allows (Lmin = 2), dense and copied rows -- every block must build (no arena
    or output overflow) and evaluate exactly."""
    rng = np.random.default_rng(11 + window + lmin)
    n = 5000
    rows = []
    for i in range(n):
        kind = i % 4
        if kind == 0:
            rows.append(sorted(set(rng.integers(0, n, 60).tolist())))          # scattered
        elif kind == 1:
            a = int(rng.integers(0, n - 200))
            rows.append(list(range(a, a + int(rng.integers(1, 150)))))          # one long run
        elif kind == 2 and i > 0:
            rows.append(sorted(set(rows[i - 1][::2] + rng.integers(0, n, 5).tolist())))  # copies with skips
        else:
            rows.append([])
    g = csr_from_rows(rows)
    params = P.BvParams(min_interval=lmin)
    _check(g, params, window=window)
