"""The device build of the BV-F layout (cmvg_create: GPU decode of the BV
stream's codes, then the shared block builder host/bvf_block.hpp on the GPU)
is bit-identical to the host build (BvStream.layout_export(kind="bvf")) --
words and block table, whole graphs and row shards -- and a device-built
handle's products, read set and statistics equal a host-built handle's
(CMVG_HOST_BUILD=1).  Reference: the A' rows of ref_matrix.hpp:13-76 taken
from the BV stream."""
import numpy as np
import pytest

import paper_1708_07271_b200 as P
from tests.helpers import bv_params, csr_from_rows, make_graph, max_rel_err, oracle_csr, x_uniform

pytestmark = pytest.mark.gpu


def _host_bvf(s, opts):
    return s.layout_export(opts, kind="bvf")


def _compare(dev_words, dev_blocks, host_words, host_blocks, b0=0, b1=None):
    hb = host_blocks[b0:b1].copy()
    off = (hb[:, 0].astype(np.uint64) | (hb[:, 1].astype(np.uint64) << np.uint64(32)))
    base = off[0]
    off -= base
    hb[:, 0] = (off & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    hb[:, 1] = (off >> np.uint64(32)).astype(np.uint32)
    assert np.array_equal(dev_blocks, hb)
    end = int(base) + len(dev_words)
    assert np.array_equal(dev_words, host_words[int(base):end])


@pytest.mark.parametrize("cfg,n,window", [(1, 1 << 16, 1536), (2, (1 << 16) + 5, 1536), (3, 1 << 15, 1536),
                                          (4, 1 << 15, 3968), (4, 20000, 256), (5, 1 << 15, 1536),
                                          (2, 9000, 256)])
def test_device_build_bit_identical(cuda, cfg, n, window):
    g = make_graph(cfg, n=n)
    s = P.BvStream.encode(g, bv_params(cfg))
    opts = P.CreateOptions(window=window)
    w, b, dev = P.BvGraph(s, opts).bvf_export()
    assert dev, "the handle's layout was not built on the device"
    hw, hb = _host_bvf(s, opts)
    _compare(w, b, hw, hb)


def test_device_build_shards_bit_identical(cuda):
    g = make_graph(2, n=(1 << 15) + 77)
    s = P.BvStream.encode(g, bv_params(2))
    hw, hb = _host_bvf(s, P.CreateOptions())
    for a, e in ((0, 8192), (8192, 20480), (20480, g.n)):
        w, b, dev = P.BvGraph(s, P.CreateOptions(row_begin=a, row_end=e)).bvf_export()
        assert dev
        _compare(w, b, hw, hb, a // 1024, (e + 1023) // 1024)


def test_device_build_edge_rows(cuda):
    rng = np.random.default_rng(5)
    n = 3000
    rows = []
    for i in range(n):
        if i % 97 == 0:
            rows.append([])
        elif i == 1500:
            rows.append(sorted(set(rng.integers(0, n, 2500).tolist())))  # hub spanning many chunks
        elif i % 5 == 1 and i > 1:
            rows.append(list(rows[i - 1]))  # exact copy: empty differential
        else:
            base = max(0, i - 40)
            rows.append(sorted(set(rng.integers(base, min(n, base + 90), 12).tolist())))
    g = csr_from_rows(rows)
    for params in (P.BvParams(), P.BvParams(max_ref=0), P.BvParams(window=1, segment_rows=2)):
        s = P.BvStream.encode(g, params)
        w, b, dev = P.BvGraph(s).bvf_export()
        assert dev
        hw, hb = _host_bvf(s, P.CreateOptions())
        _compare(w, b, hw, hb)
    for rows in ([[]], [[0]], [[], [1], [0, 1]]):
        s = P.BvStream.encode(csr_from_rows(rows), P.BvParams())
        w, b, dev = P.BvGraph(s).bvf_export()
        hw, hb = _host_bvf(s, P.CreateOptions())
        _compare(w, b, hw, hb)


def test_device_and_host_built_handles_agree(cuda, monkeypatch):
    import torch

    g = make_graph(2, n=1 << 16)
    s = P.BvStream.encode(g, bv_params(2))
    x = x_uniform(g.n, 4)
    dd = P.BvGraph(s)
    monkeypatch.setenv("CMVG_HOST_BUILD", "1")
    dh = P.BvGraph(s)
    monkeypatch.delenv("CMVG_HOST_BUILD")
    assert dd.bvf_export()[2] and not dh.bvf_export()[2]
    yd, yh = dd.matvec(x), dh.matvec(x)
    assert np.array_equal(yd, yh)  # identical layouts: identical sums
    assert max_rel_err(yd, oracle_csr(g).matvec(x)) <= 1e-12
    assert np.array_equal(dd.read_set(), dh.read_set())
    idd, idh = dd.info(), dh.info()
    for k in ("bvf_stream_bytes", "bvf_terms", "bvf_pad_terms", "bvf_slot_terms", "bvf_esc_terms", "bvf_esc_blocks",
              "bvf_max_K", "bvf_min_cbits", "max_depth", "adds_per_product"):
        assert idd[k] == idh[k], k
    assert abs(idd["window_coverage"] - idh["window_coverage"]) < 1e-12
    # fp32 product and PageRank step through the device-built handle
    y32 = dd.matvec(x.astype(np.float32))
    want32 = oracle_csr(g).matvec(x.astype(np.float32).astype(np.float64))
    assert max_rel_err(y32, want32) <= 1e-5
    del torch


def test_device_build_rejects_corrupt_stream(cuda):
    g = make_graph(1, n=1 << 12)
    s = P.BvStream.encode(g, bv_params(1))
    w = s.words()
    w[len(w) // 2] ^= 0xFFFF0000
    bad = P.BvStream.from_words(g.n, g.m, s.params, w, s.stats()["stream_bits"], s.segment_offsets())
    with pytest.raises(P.CorruptionError):
        P.BvGraph(bad)
