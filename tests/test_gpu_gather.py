"""GPU parity of the gather product y = A x^T (the hot path) against the
oracle's matvec_csr (csr.hpp:48-55) and matvec_ref on compress(g, 7)
(ref_matvec.hpp:30-35).  Tolerances (BASELINE.json north_star): fp64 1e-12
relative per entry, fp32 1e-5 relative per entry against fp64 matvec_csr on the
fp32-rounded x; empty rows exactly 0."""
import numpy as np
import pytest

import paper_1708_07271_b200 as P
from oracle import pyoracle as O
from tests.helpers import bv_params, csr_from_rows, make_graph, max_rel_err, oracle_csr, x_uniform

pytestmark = pytest.mark.gpu

F64_TOL = 1e-12
F32_TOL = 1e-5


def check_gather(g, params, opts=None, seed=1, dtype=np.float64, device=False):
    import torch

    s = P.BvStream.encode(g, params)
    dg = P.BvGraph(s, opts or P.CreateOptions())
    x = x_uniform(g.n, seed)
    ref = oracle_csr(g)
    if dtype == np.float32:
        x32 = x.astype(np.float32)
        want = ref.matvec(x32.astype(np.float64), 8)
        if device:
            y = dg.matvec(torch.from_numpy(x32).cuda()).cpu().numpy()
        else:
            y = dg.matvec(x32)
        err = max_rel_err(y, want)
        assert err <= F32_TOL, err
    else:
        want = ref.matvec(x, 8)
        if device:
            y = dg.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
        else:
            y = dg.matvec(x)
        err = max_rel_err(y, want)
        assert err <= F64_TOL, err
    return dg, s, x, y


@pytest.mark.parametrize("mode", ["prefix", "direct"])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_gather_copy_model_small(cuda, mode, dtype):
    g = make_graph(1, n=1 << 16)
    check_gather(g, bv_params(1), P.CreateOptions(interval_mode=mode), dtype=dtype)


def test_gather_device_pointers(cuda):
    g = make_graph(2, n=1 << 17)
    check_gather(g, bv_params(2), device=True)
    check_gather(g, bv_params(2), dtype=np.float32, device=True)


def test_gather_matches_matvec_ref(cuda):
    g = make_graph(1, n=1 << 15)
    s = P.BvStream.encode(g, bv_params(1))
    dg = P.BvGraph(s)
    x = x_uniform(g.n, 3)
    rm = O.RefMatrix.compress(oracle_csr(g), 7)
    want, _ = rm.matvec(x)
    assert max_rel_err(dg.matvec(x), want) <= F64_TOL


@pytest.mark.parametrize("lanes,block_rows,window", [(256, 1024, 2048), (256, 1024, 1536), (256, 1024, 1024), (256, 1024, 3968),
                                                      (256, 1024, 512), (256, 1024, 128)])
def test_gather_layout_variants(cuda, lanes, block_rows, window):
    g = make_graph(2, n=(1 << 16) + 777)  # ragged last block
    check_gather(g, bv_params(2), P.CreateOptions(lanes=lanes, block_rows=block_rows, window=window))


def test_gather_stream_from_global(cuda):
    # tiny smem cap: every block decodes straight from global memory
    g = make_graph(1, n=1 << 15)
    check_gather(g, bv_params(1), P.CreateOptions(stream_cap_words=16))


def test_gather_unbounded_chains_social(cuda):
    g = make_graph(4, n=1 << 16)
    dg, s, _, _ = check_gather(g, bv_params(4), dtype=np.float32)
    assert s.stats()["max_depth"] > 3


def test_gather_long_copy_chain(cuda):
    # every row equals row 0 -> chain depth up to the segment length (R=0)
    n, base = 4096, 40
    rows = [list(range(0, 2 * base, 2))] * n
    g = csr_from_rows(rows)
    check_gather(g, P.BvParams(max_ref=0))
    check_gather(g, P.BvParams(max_ref=3))


def test_gather_edge_cases(cuda):
    # empty rows, self loops, a single row, columns at 0 and n-1, long intervals
    cases = [
        [[]],
        [[0]],
        [[], [], []],
        [[0, 1, 2, 3, 4, 5, 6, 7, 8, 9], [], [9], [0, 9]] + [[]] * 6,
        [list(range(0, 3000)), list(range(1, 3001)), [2999, 3000], list(range(5, 3001, 2))] + [[]] * 2997,
    ]
    for rows in cases:
        g = csr_from_rows(rows)
        check_gather(g, P.BvParams())
        check_gather(g, P.BvParams(), dtype=np.float32)


def test_gather_far_columns(cuda):
    # columns far outside every block's x-window -> global-memory gathers and intervals
    rng = np.random.default_rng(4)
    n = 50_000
    rows = []
    for i in range(n):
        k = int(rng.integers(0, 12))
        c = set(rng.integers(0, n, size=k).tolist())
        if rng.random() < 0.2:
            s0 = int(rng.integers(0, n - 20))
            c.update(range(s0, s0 + 8))
        rows.append(sorted(c))
    g = csr_from_rows(rows)
    check_gather(g, P.BvParams())


def test_gather_shards_cover_rows(cuda):
    g = make_graph(1, n=(1 << 16) + 100)
    s = P.BvStream.encode(g, bv_params(1))
    x = x_uniform(g.n, 5)
    want = oracle_csr(g).matvec(x, 8)
    bounds = [0, 16384, 32768, g.n]
    parts = []
    for a, b in zip(bounds[:-1], bounds[1:]):
        dg = P.BvGraph(s, P.CreateOptions(row_begin=a, row_end=b))
        parts.append(dg.matvec(x))
    assert max_rel_err(np.concatenate(parts), want) <= F64_TOL


def test_gather_bad_options(cuda):
    g = make_graph(1, n=4096)
    s = P.BvStream.encode(g, bv_params(1))
    with pytest.raises(ValueError):
        P.BvGraph(s, P.CreateOptions(lanes=96))
    with pytest.raises(ValueError):
        P.BvGraph(s, P.CreateOptions(lanes=128, block_rows=1024))


def test_gather_dimension_errors(cuda):
    g = make_graph(1, n=4096)
    dg = P.BvGraph(P.BvStream.encode(g, bv_params(1)))
    with pytest.raises(ValueError):
        dg.matvec(np.zeros(4095))


def test_adds_per_product(cuda):
    g = make_graph(1, n=1 << 14)
    dg = P.BvGraph(P.BvStream.encode(g, bv_params(1)))
    assert 0 < dg.adds_per_product() < g.m
    assert dg.dimension() == g.n


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_gather_multi_unit_and_heavy_rows(cuda, dtype):
    # rows split across adjacent lanes of multi slices (segmented warp
    # reduction) and rows beyond 32 units (warp path), mixed with light rows
    rng = np.random.default_rng(5)
    n = 4096

    def row(k):
        if k % 97 == 0:
            return sorted(set(rng.integers(0, n, 700).tolist()))
        if k % 5 == 0:
            return sorted(set(rng.integers(max(0, k - 3000), min(n, k + 3000), 120).tolist()))
        if k % 7 == 0:
            return list(range(max(0, k - 40), min(n, k + 40), 2))  # 40 points near the diagonal
        return sorted(set(rng.integers(0, n, 3).tolist()))
    g = csr_from_rows([row(k) for k in range(n)])
    check_gather(g, P.BvParams(), dtype=dtype)
    check_gather(g, P.BvParams(), P.CreateOptions(window=512), dtype=dtype)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("cfg,n,window", [(2, (1 << 17) + 333, 1536), (4, 1 << 15, 1536), (2, 1 << 16, 256)])
def test_gather_host_pinned_pipelined(cuda, dtype, cfg, n, window):
    # pinned host x / y take the pipelined path (chunked H2D, blocks launched as
    # their window arrives, far columns read from mapped host memory, chunked
    # D2H); pageable buffers the plain path -- both must match the oracle
    import torch

    g = make_graph(cfg, n=n)
    dg = P.BvGraph(P.BvStream.encode(g, bv_params(cfg)), P.CreateOptions(window=window))
    x = x_uniform(g.n, 5).astype(dtype)
    want = oracle_csr(g).matvec(x.astype(np.float64), 8)
    tol = F64_TOL if dtype == np.float64 else F32_TOL
    xp = torch.from_numpy(x).pin_memory()
    yp = torch.empty(g.n, dtype=xp.dtype).pin_memory()
    yn = yp.numpy()
    for _ in range(2):
        yn[:] = np.nan
        dg.matvec(xp.numpy(), yn)
        assert max_rel_err(yn, want) <= tol
    assert max_rel_err(dg.matvec(x), want) <= tol


def test_gather_host_pinned_pipelined_shard(cuda):
    # a row shard (not starting at 0) on the pipelined host path: y holds the
    # shard's rows; x is the full vector
    import torch

    g = make_graph(2, n=(1 << 17) + 99)
    s = P.BvStream.encode(g, bv_params(2))
    a, b = 32768, g.n
    dg = P.BvGraph(s, P.CreateOptions(row_begin=a, row_end=b))
    x = x_uniform(g.n, 6)
    want = oracle_csr(g).matvec(x, 8)[a:b]
    xp = torch.from_numpy(x).pin_memory()
    yp = torch.empty(b - a, dtype=torch.float64).pin_memory()
    dg.matvec(xp.numpy(), yp.numpy())
    assert max_rel_err(yp.numpy(), want) <= F64_TOL


@pytest.mark.parametrize("n,shard", [(20000, False), ((1 << 16) + 7, False), ((1 << 17) + 99, True)])
def test_gather_host_pageable_staged(cuda, n, shard):
    # pageable host x / y (numpy, std::vector spans): the same pipeline through
    # the handle's pinned staging buffers, host copies overlapped with the
    # transfers; n = 20000 has 20 blocks (an empty last pipeline chunk)
    g = make_graph(2, n=n)
    s = P.BvStream.encode(g, bv_params(2))
    a, b = (32768, g.n) if shard else (0, g.n)
    dg = P.BvGraph(s, P.CreateOptions(row_begin=a, row_end=b))
    for dtype, tol in ((np.float64, F64_TOL), (np.float32, F32_TOL)):
        x = x_uniform(g.n, 7).astype(dtype)
        want = oracle_csr(g).matvec(x.astype(np.float64), 8)[a:b]
        y = np.full(b - a, np.nan, dtype=dtype)
        for _ in range(2):
            dg.matvec(x, y)
            assert max_rel_err(y, want) <= tol
            y[:] = np.nan


@pytest.mark.parametrize("deg", [3.0, 12.0, 40.0, 150.0])
def test_csr_baseline_matches_oracle(cuda, deg):
    """The uncompressed comparison kernel (matvec_csr on the GPU, csr.hpp:48-55)
    against the oracle, for every sub-warp width it picks by mean degree."""
    import torch

    g = P.CsrGraph.copy_model((1 << 14) + 3, deg, seed=5)  # a partial last block of rows
    x = x_uniform(g.n, 3)
    want = oracle_csr(g).matvec(x, 8)
    ro = torch.from_numpy(g.row_offsets.astype(np.int64)).cuda()
    co = torch.from_numpy(g.columns.view(np.int32)).cuda()
    y = P.csr_matvec_device(ro, co, torch.from_numpy(x).cuda()).cpu().numpy()
    assert max_rel_err(y, want) <= F64_TOL
    assert np.all(y[want == 0] == 0)
    e = P.csr_matvec_device(torch.zeros(1, dtype=torch.int64, device="cuda"),
                            torch.zeros(0, dtype=torch.int32, device="cuda"),
                            torch.zeros(0, dtype=torch.float64, device="cuda"))
    assert e.numel() == 0  # n = 0


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_gather_hub_rows_split_into_items(cuda, dtype):
    """Rows far beyond 32 units are cut into 512-point work items taken by any
    warp and combined in item order (bvs_heavy / bvs_heavy_finish): hub rows of
    several items, with intervals and a reference, plus ordinary rows."""
    rng = np.random.default_rng(21)
    n = 6000
    rows = []
    for i in range(n):
        if i % 997 == 5:  # hub: thousands of random columns plus a run (interval)
            cols = set(rng.choice(n, size=int(rng.integers(1500, 4000)), replace=False).tolist())
            cols.update(range(100, 140))
        elif i % 997 == 6:  # references the hub above (copy with deletions)
            cols = set(c for c in rows[i - 1] if rng.random() < 0.7)
        else:
            cols = set((i + rng.geometric(1 / 40, size=int(rng.integers(0, 25)))) % n)
        rows.append(sorted(cols))
    g = csr_from_rows(rows)
    dg, s, _, _ = check_gather(g, bv_params(2), dtype=dtype)
    assert dg.info()["bvf_max_K"] > 16  # the hubs' blocks get wide chunks (spread over all threads)
    check_gather(g, bv_params(2), dtype=dtype, device=True)


def test_gather_from_loaded_container(cuda, tmp_path):
    """A BV stream written to and read back from a CBV1 container drives the
    device handle exactly like the encoder's stream."""
    g = P.CsrGraph.copy_model(1 << 13, 12.0, seed=31)
    s = P.BvStream.encode(g, P.BvParams())
    p = tmp_path / "g.cbv"
    s.save(str(p))
    t = P.BvStream.load(str(p))
    x = x_uniform(g.n, 9)
    y0 = P.BvGraph(s).matvec(x)
    y1 = P.BvGraph(t).matvec(x)
    assert np.array_equal(y0, y1)
    assert max_rel_err(y1, oracle_csr(g).matvec(x, 8)) <= F64_TOL


def test_gather_hub_rows_concurrent_streams(cuda):
    """Hub rows (spread over all chunks of their block) on a handle serving
    concurrent products on distinct streams (cmvg.h contract)."""
    import torch

    g = P.CsrGraph.social(1 << 15, seed=77)
    dg = P.BvGraph(P.BvStream.encode(g, P.BvParams(max_ref=0)))
    assert dg.info()["bvf_max_K"] > 16
    xs = [torch.from_numpy(x_uniform(g.n, s)).cuda() for s in (1, 2, 3, 4)]
    want = [dg.matvec(x).cpu().numpy() for x in xs]
    streams = [torch.cuda.Stream() for _ in xs]
    ys = [torch.empty_like(x) for x in xs]
    for _ in range(3):
        for x, y, st in zip(xs, ys, streams):
            with torch.cuda.stream(st):
                dg.matvec(x, y, stream=st.cuda_stream)
        torch.cuda.synchronize()
        for y, w in zip(ys, want):
            assert np.array_equal(y.cpu().numpy(), w)
    ref = oracle_csr(g)
    for x, w in zip(xs, want):
        assert max_rel_err(w, ref.matvec(x.cpu().numpy(), 8)) <= F64_TOL


def test_gather_window_bulk_copy_and_fallbacks(cuda):
    """fp64 products at the default shape take the x-window by a TMA bulk copy
    (the ABI's 16-byte aligned device buffers, whole window in range); windows
    cut by the end of the graph take the per-thread path.  Both fill the same
    table: wide-range values, a graph whose last windows run past n, and the
    device- and host-pointer calls must agree bit for bit."""
    import torch

    for n in ((1 << 16) + 517, 1 << 16, 1536 + 3):  # last window past n; all windows whole; a single cut window
        g = make_graph(2, n=n)
        s = P.BvStream.encode(g, bv_params(2))
        dg = P.BvGraph(s, P.CreateOptions())
        ref = oracle_csr(g)
        x = x_uniform(n, 5)
        x[::97] *= 2.0**-40  # wide dynamic range inside every window (block grid split)
        want = ref.matvec(x, 8)
        xd = torch.from_numpy(x).cuda()
        yd = torch.empty_like(xd)
        dg.matvec(xd, yd)
        y = yd.cpu().numpy()
        assert max_rel_err(y, want) <= F64_TOL
        assert np.array_equal(dg.matvec(x), y)
