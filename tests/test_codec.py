"""CPU tests of the host side: generators, the canonical BV codec (encode ->
decode round trip, corruption detection), the BV-D device-layout builder
(re-decoded with the kernels' arithmetic in tests/layout_ref.py), and the
C-ABI surface (library loads and exports every symbol include/cmvg.h declares)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1708_07271_b200 as P
from tests.helpers import CONFIGS, bv_params, csr_from_rows, make_graph
from tests.layout_ref import decode_layout, decode_sliced, scatter_bvt_int

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_abi_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "cmvg.h")).read()
    names = set(re.findall(r"\b(cmvg_[a-z0-9_]+)\s*\(", hdr))
    lib = P.load_library()
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    assert set(P.EXPORTED_SYMBOLS) <= names


def rows_of(g):
    ro, co = g.row_offsets, g.columns
    return [co[ro[u]:ro[u + 1]].tolist() for u in range(g.n)]


def test_generator_deterministic_and_degree():
    a = make_graph(1, n=1 << 16)
    b = make_graph(1, n=1 << 16)
    assert np.array_equal(a.row_offsets, b.row_offsets) and np.array_equal(a.columns, b.columns)
    assert abs(a.m / a.n - 12.0) / 12.0 < 0.03
    ro, co = a.row_offsets, a.columns
    for u in range(0, a.n, 997):  # rows sorted, strict, in range
        r = co[ro[u]:ro[u + 1]]
        assert np.all(np.diff(r.astype(np.int64)) > 0) and (r.size == 0 or r[-1] < a.n)


def test_social_generator():
    g = make_graph(4, n=1 << 16)
    deg = g.out_degrees()
    assert deg.min() >= 1 and 20 < deg.mean() < 40


@pytest.mark.parametrize("cfg,n", [(1, 1 << 15), (2, 20000), (4, 1 << 14)])
@pytest.mark.parametrize("seg", [1024, 64])
def test_bv_roundtrip(cfg, n, seg):
    g = make_graph(cfg, n=n)
    s = P.BvStream.encode(g, bv_params(cfg, segment_rows=seg))
    st = s.stats()
    assert st["stream_bits"] > 0
    if CONFIGS[cfg]["R"]:
        assert st["max_depth"] <= CONFIGS[cfg]["R"]
    assert st["copied_edges"] + st["interval_edges"] + st["residual_edges"] == g.m
    h = s.decode_host()
    assert np.array_equal(h.row_offsets, g.row_offsets) and np.array_equal(h.columns, g.columns)


def test_bv_roundtrip_random_small():
    rng = np.random.default_rng(3)
    for _ in range(60):
        n = int(rng.integers(1, 300))
        dens = rng.uniform(0.0, 0.3)
        A = rng.random((n, n)) < dens
        rows = [np.nonzero(A[u])[0].tolist() for u in range(n)]
        g = csr_from_rows(rows)
        for params in (P.BvParams(), P.BvParams(max_ref=0), P.BvParams(window=1, segment_rows=4),
                       P.BvParams(window=3, max_ref=1, min_interval=2, segment_rows=16)):
            h = P.BvStream.encode(g, params).decode_host()
            assert rows_of(h) == rows


def test_bv_words_roundtrip_and_corruption():
    g = make_graph(1, n=1 << 12)
    s = P.BvStream.encode(g, bv_params(1))
    w, seg, nbits = s.words(), s.segment_offsets(), s.stats()["stream_bits"]
    s2 = P.BvStream.from_words(g.n, g.m, s.params, w, nbits, seg)
    assert rows_of(s2.decode_host()) == rows_of(g)
    bad = w.copy()
    bad[len(bad) // 3] ^= 0x00F0F000
    with pytest.raises((P.CorruptionError, ValueError, IndexError)):
        P.BvStream.from_words(g.n, g.m, s.params, bad, nbits, seg).decode_host()
    with pytest.raises((P.CorruptionError, ValueError, IndexError)):
        P.BvStream.from_words(g.n, g.m, s.params, w[: len(w) // 2], nbits // 2, seg).decode_host()


def test_bv_params_validation():
    g = make_graph(1, n=256)
    with pytest.raises(ValueError):
        P.BvStream.encode(g, P.BvParams(zeta_k=1))
    with pytest.raises(ValueError):
        P.BvStream.encode(g, P.BvParams(min_interval=1))


@pytest.mark.parametrize("cfg,n,window", [(1, 5000, 1536), (2, 9000, 2048), (4, 3000, 1536)])
def test_device_layout_decodes_to_adjacency(cfg, n, window):
    g = make_graph(cfg, n=n)
    s = P.BvStream.encode(g, bv_params(cfg))
    words, blocks = s.layout_export(P.CreateOptions(block_rows=1024, window=window))
    refs, rows = decode_layout(words, blocks, g.n, 1024, 4, W=window)
    assert rows == rows_of(g)


@pytest.mark.parametrize("cfg,n,window", [(1, 5000, 1536), (2, 9000, 2048), (3, 6000, 1536), (4, 3000, 1536)])
def test_sliced_layout_decodes_to_adjacency(cfg, n, window):
    g = make_graph(cfg, n=n)
    s = P.BvStream.encode(g, bv_params(cfg))
    words, blocks = s.layout_export(P.CreateOptions(block_rows=1024, window=window), sliced=True)
    refs, rows = decode_sliced(words, blocks, g.n, 1024, 4, W=window)
    assert rows == rows_of(g)
    info = s.layout_info(P.CreateOptions(block_rows=1024, window=window))
    assert info["bvs_lane_iters_used"] <= info["bvs_lane_iters"]


def test_device_layout_escapes_and_edge_rows():
    # heavy rows force the escape table; empty rows and far columns too
    n = 3000
    rows = [[] for _ in range(n)]
    rows[5] = list(range(0, 3000, 3))           # 1000 residual-ish entries
    rows[6] = list(range(0, 3000, 3))[:-7]      # references row 5, many minus? no: subset
    rows[7] = list(range(100, 2900))            # one long interval
    rows[8] = sorted(set(range(0, 3000, 7)) | set(range(1000, 1100)))
    rows[2999] = [0, 2999]
    g = csr_from_rows(rows)
    s = P.BvStream.encode(g, P.BvParams())
    words, blocks = s.layout_export(P.CreateOptions(block_rows=1024, window=512))
    _, got = decode_layout(words, blocks, n, 1024, 4, W=512)
    assert got == rows
    words, blocks = s.layout_export(P.CreateOptions(block_rows=1024, window=512), sliced=True)
    _, got = decode_sliced(words, blocks, n, 1024, 4, W=512)
    assert got == rows


def test_layout_info_sizes():
    g = make_graph(2, n=1 << 16)
    s = P.BvStream.encode(g, bv_params(2))
    li = s.layout_info()
    S = s.stats()["stream_bits"]
    assert li["bvd_stream_bytes"] * 8 >= li["bvd_row_bits"]
    assert 1.0 <= li["bvd_row_bits"] / S < 2.0
    assert li["window_coverage"] > 0.99
    assert li["max_depth"] <= 3


def test_sliced_layout_multi_and_heavy_rows():
    # rows of ~120 scattered columns need 8 units (adjacent lanes of a multi
    # slice); rows of ~700 need > 32 units and take the warp (heavy) path
    rng = np.random.default_rng(5)
    n = 2048
    def row(k):
        if k % 97 == 0:
            return sorted(set(rng.integers(0, n, 700).tolist()))
        if k % 5 == 0:
            return sorted(set(rng.integers(0, n, 120).tolist()))
        return sorted(set(rng.integers(0, n, 3).tolist()))
    rows = [row(k) for k in range(n)]
    g = csr_from_rows(rows)
    s = P.BvStream.encode(g, P.BvParams())
    words, blocks = s.layout_export(P.CreateOptions(block_rows=1024, window=1536), sliced=True)
    _, got = decode_sliced(words, blocks, n, 1024, 4, W=1536)
    assert got == rows
    info = s.layout_info()
    assert info["bvs_heavy_rows"] > 0


@pytest.mark.parametrize("cfg,n,window", [(1, 5000, 1536), (2, 9000, 1536), (4, 3000, 1536), (2, 4000, 256)])
def test_target_layout_scatter_exact(cfg, n, window):
    g = make_graph(cfg, n=n)
    s = P.BvStream.encode(g, bv_params(cfg))
    words, blocks = s.layout_export(P.CreateOptions(block_rows=1024, window=window), kind="bvt")
    x = np.random.default_rng(3).integers(0, 1000, g.n)
    want = np.zeros(g.n, dtype=np.int64)
    ro, co = g.row_offsets, g.columns
    for i in range(g.n):
        want[co[ro[i]:ro[i + 1]]] += x[i]
    assert np.array_equal(scatter_bvt_int(words, blocks, g.n, 1024, window, x), want)


def test_target_layout_heavy_targets():
    # no references (w = 0): every row hits column 7 -> > 512 entries per block
    rng = np.random.default_rng(11)
    n = 3000
    rows = [sorted({7} | set(rng.integers(0, n, 3).tolist())) for _ in range(n)]
    g = csr_from_rows(rows)
    s = P.BvStream.encode(g, P.BvParams(window=0))
    assert s.layout_info()["bvt_heavy_targets"] > 0
    words, blocks = s.layout_export(kind="bvt")
    x = rng.integers(0, 1000, n)
    want = np.zeros(n, dtype=np.int64)
    for i, r in enumerate(rows):
        want[r] += x[i]
    assert np.array_equal(scatter_bvt_int(words, blocks, n, 1024, 1536, x), want)


def test_compression_stats():
    """cmv::stats mirror (ref_matrix.hpp:78-89) on a BV stream: A' = minus
    entries + extra entries; without references A' = A and the ratio is 1."""
    g = make_graph(2, n=1 << 13)
    s = P.BvStream.encode(g, P.BvParams())
    st, c = s.stats(), P.compression_stats(s)
    assert c.n == g.n and c.m == g.m
    assert c.m_prime == g.m - st["copied_edges"] + st["minus_edges"]
    assert c.m_prime < c.m and abs(c.ratio - c.m / c.m_prime) < 1e-12 and not c.ratio_by_convention
    assert c.rows_self_coded == g.n - st["rows_with_ref"] and c.max_chain == st["max_depth"]
    c0 = P.compression_stats(P.BvStream.encode(g, P.BvParams(window=0)))
    assert c0.m_prime == g.m and c0.ratio == 1.0 and c0.rows_self_coded == g.n and c0.max_chain == 0
    e = P.compression_stats(P.BvStream.encode(csr_from_rows([[]] * 5),
                                              P.BvParams()))
    assert e.m_prime == 0 and e.ratio == 1.0 and e.ratio_by_convention


@pytest.mark.parametrize("cfg,n,seg", [(1, 5000, 1024), (4, 3000, 1024), (2, 4000, 7)])
def test_reconstruct_row_random_access(cfg, n, seg):
    """reconstruct_row (ref_matrix.hpp:71-73): any row from the stream alone,
    bit-exact; out_of_range past n (IndexError), also through the C ABI."""
    g = make_graph(cfg, n=n)
    s = P.BvStream.encode(g, bv_params(cfg) if seg == 1024 else P.BvParams(segment_rows=seg))
    rows = rows_of(g)
    rng = np.random.default_rng(cfg)
    for i in list(rng.integers(0, n, 60)) + [0, n - 1, seg - 1, min(seg, n - 1)]:
        assert s.reconstruct_row(int(i)).tolist() == rows[int(i)]
    with pytest.raises(IndexError):
        s.reconstruct_row(n)
    lib = P.load_library()
    d = ctypes.c_uint64()
    assert lib.cmvg_bv_reconstruct_row(s._h, n, None, 0, ctypes.byref(d)) == 2  # CMVG_ERR_RANGE
