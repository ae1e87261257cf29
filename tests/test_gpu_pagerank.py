"""Device PageRank (pagerank.hpp:83-102) on BV(A^T) against the oracle's
pagerank with CsrKernel(A^T): per-entry relative error <= 1e-12, sum p = 1
within 1e-10, both dangling policies, early stop on the L1
tolerance, and the per-shard step used by the multi-GPU driver."""
import json
import os

import numpy as np
import pytest

import paper_1708_07271_b200 as P
from oracle import pyoracle as O
from tests.helpers import csr_from_rows, make_graph

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def bv_of_transpose(g: P.CsrGraph, **kw):
    return P.BvStream.encode(g.transpose(), P.BvParams(**kw))


def oracle_pr(g: P.CsrGraph, **kw):
    og = O.Csr.from_arrays(g.n, g.row_offsets, g.columns)
    return O.pagerank_csr(og.transpose(), og.out_degrees(), **kw)


def rel(a, b):
    return float(np.max(np.abs(a - b) / np.abs(b)))


@pytest.mark.parametrize("e", GOLD["pagerank"], ids=lambda e: e["spec"])
def test_pagerank_golden(cuda, e):
    rows = [[] for _ in range(e["n"])]
    for u, v in e["edges"]:
        rows[u].append(v)
    g = csr_from_rows([sorted(r) for r in rows])
    k = P.BvGpuKernel(P.BvGraph(bv_of_transpose(g)))
    res = P.pagerank(k, g.out_degrees(), P.PageRankConfig(alpha=e["alpha"], iterations=e["iterations"]))
    assert res.iterations_run == e["iterations"]
    assert np.max(np.abs(res.ranks - np.asarray(e["want"]))) <= e["tol"]


@pytest.mark.parametrize("dangling", ["uniform", "drop"])
def test_pagerank_matches_oracle(cuda, dangling):
    g = make_graph(3, n=1 << 16)  # copy model, mean degree 24 (config 3 shape); has dangling rows
    assert (g.out_degrees() == 0).any()
    dg = P.BvGraph(bv_of_transpose(g))
    p, it = dg.pagerank(g.out_degrees(), alpha=0.15, iterations=50, dangling=dangling)
    want, wit = oracle_pr(g, alpha=0.15, iterations=50, dangling=dangling)
    assert it == wit == 50
    assert rel(p, want) <= 1e-12
    if dangling == "uniform":
        assert abs(p.sum() - 1.0) <= 1e-10


def test_pagerank_l1_tolerance(cuda):
    g = make_graph(3, n=1 << 14)
    dg = P.BvGraph(bv_of_transpose(g))
    p, it = dg.pagerank(g.out_degrees(), iterations=200, l1_tolerance=1e-10)
    want, wit = oracle_pr(g, iterations=200, l1_tolerance=1e-10)
    assert it == wit < 200
    assert rel(p, want) <= 1e-12


def test_pagerank_device_buffers_and_errors(cuda):
    import torch

    g = make_graph(3, n=1 << 14)
    dg = P.BvGraph(bv_of_transpose(g))
    deg = torch.from_numpy(g.out_degrees().astype(np.int32)).cuda()
    p, it = dg.pagerank(deg, iterations=20)
    want, _ = oracle_pr(g, iterations=20)
    assert rel(p.cpu().numpy(), want) <= 1e-12
    k = P.BvGpuKernel(dg)
    with pytest.raises(ValueError):
        P.pagerank(k, g.out_degrees(), P.PageRankConfig(alpha=1.5))
    with pytest.raises(ValueError):
        P.pagerank(k, g.out_degrees(), P.PageRankConfig(iterations=0))
    with pytest.raises(ValueError):
        P.pagerank(k, g.out_degrees()[:-1])


def test_pagerank_shard_steps(cuda):
    """Two row shards of A^T on one GPU, exchanged by hand exactly as the
    multi-GPU driver does (all_gather of q, sum of the partials)."""
    import torch

    from paper_1708_07271_b200.distributed import plan_shards

    g = make_graph(3, n=(1 << 15) + 300)
    n = g.n
    s = bv_of_transpose(g)
    plan = plan_shards(n, 2, 1024)
    deg = torch.from_numpy(g.out_degrees().astype(np.int32)).cuda()
    shards = []
    for r in range(2):
        a, b = plan.bounds(r)
        shards.append((a, b, P.BvGraph(s, P.CreateOptions(row_begin=a, row_end=b))))
    p = torch.full((n,), 1.0 / n, dtype=torch.float64, device="cuda")
    q = torch.where(deg > 0, p / deg.clamp(min=1).double(), torch.zeros_like(p))
    dmass = float(p[deg == 0].sum())
    for _ in range(30):
        p_next, q_next = torch.empty_like(p), torch.empty_like(q)
        tot = torch.zeros(2, dtype=torch.float64, device="cuda")
        for a, b, dgs in shards:
            part = torch.zeros(2, dtype=torch.float64, device="cuda")
            dgs.pagerank_step(q, deg[a:b], 0.15, dmass, "uniform", p[a:b], p_next[a:b], q_next[a:b], part)
            tot += part
        p, q = p_next, q_next
        dmass = float(tot[0])
    want, _ = oracle_pr(g, iterations=30)
    assert rel(p.cpu().numpy(), want) <= 1e-12


def test_pagerank_shard_steps_device_dmass(cuda):
    """cmvg_pagerank_step_dev: the dangling mass is read from device memory
    (the previous step's summed partials), so no value crosses to the host
    between iterations; three shards on one GPU, 40 iterations, no sync."""
    import torch

    from paper_1708_07271_b200.distributed import plan_shards

    g = make_graph(3, n=(1 << 15) + 4000)
    n = g.n
    s = bv_of_transpose(g)
    plan = plan_shards(n, 3, 1024)
    deg = torch.from_numpy(g.out_degrees().astype(np.int32)).cuda()
    shards = [(a, b, P.BvGraph(s, P.CreateOptions(row_begin=a, row_end=b)))
              for a, b in (plan.bounds(r) for r in range(3))]
    p = torch.full((n,), 1.0 / n, dtype=torch.float64, device="cuda")
    q = torch.where(deg > 0, p / deg.clamp(min=1).double(), torch.zeros_like(p))
    tot = torch.zeros(2, dtype=torch.float64, device="cuda")
    tot[0] = p[deg == 0].sum()
    parts = torch.zeros((3, 2), dtype=torch.float64, device="cuda")
    for _ in range(40):
        p_next, q_next = torch.empty_like(p), torch.empty_like(q)
        for r, (a, b, dgs) in enumerate(shards):
            dgs.pagerank_step_dev(q, deg[a:b], 0.15, tot, "uniform", p[a:b], p_next[a:b], q_next[a:b], parts[r])
        tot = parts.sum(0)  # the all_reduce of the multi-GPU driver
        p, q = p_next, q_next
    want, _ = oracle_pr(g, iterations=40)
    assert rel(p.cpu().numpy(), want) <= 1e-12
    assert abs(float(p.sum()) - 1.0) <= 1e-10


@pytest.mark.parametrize("window", [1536, 256])
def test_pagerank_shard_steps_halo_read_set(cuda, window):
    """Each shard's step sees q only at its own rows and its read_set() (every
    other entry NaN): the halo exchange's contract.  Results must match the
    oracle, and the halo must be much smaller than the full vector."""
    import torch

    from paper_1708_07271_b200.distributed import plan_shards

    g = make_graph(3, n=(1 << 16) + 300)
    n = g.n
    s = bv_of_transpose(g)
    plan = plan_shards(n, 3, 1024)
    deg = torch.from_numpy(g.out_degrees().astype(np.int32)).cuda()
    shards = []
    for r in range(3):
        a, b = plan.bounds(r)
        dgs = P.BvGraph(s, P.CreateOptions(row_begin=a, row_end=b, window=window))
        rs = torch.from_numpy(dgs.read_set().astype(np.int64)).cuda()
        keep = torch.zeros(n, dtype=torch.bool, device="cuda")
        keep[a:b] = True
        keep[rs] = True
        halo = int(keep.sum()) - (b - a)
        assert halo < n // 2
        shards.append((a, b, dgs, keep))
    p = torch.full((n,), 1.0 / n, dtype=torch.float64, device="cuda")
    q = torch.where(deg > 0, p / deg.clamp(min=1).double(), torch.zeros_like(p))
    dmass = float(p[deg == 0].sum())
    nan = torch.full_like(q, float("nan"))
    for _ in range(20):
        p_next, q_next = torch.empty_like(p), torch.empty_like(q)
        tot = torch.zeros(2, dtype=torch.float64, device="cuda")
        for a, b, dgs, keep in shards:
            part = torch.zeros(2, dtype=torch.float64, device="cuda")
            dgs.pagerank_step(torch.where(keep, q, nan), deg[a:b], 0.15, dmass, "uniform", p[a:b], p_next[a:b],
                              q_next[a:b], part)
            tot += part
        p, q = p_next, q_next
        dmass = float(tot[0])
    want, _ = oracle_pr(g, iterations=20)
    assert rel(p.cpu().numpy(), want) <= 1e-12


def test_pagerank_shard_steps_fused_push(cuda):
    """The fused exchange (cmvg_pagerank_step_push): three shards on one GPU,
    each with its own pair of q buffers; a shard's kernel writes its q' rows
    locally and stores them into the buffers of the shards whose read set
    holds them (here plain local buffers stand in for NVLink peer memory --
    the kernel only sees pointers).  Nothing else moves q; every entry outside
    a shard's rows and read set stays NaN."""
    import torch

    from paper_1708_07271_b200.distributed import plan_shards

    g = make_graph(3, n=(1 << 16) + 300)
    n = g.n
    s = bv_of_transpose(g)
    world = 3
    plan = plan_shards(n, world, 1024)
    deg = torch.from_numpy(g.out_degrees().astype(np.int32)).cuda()
    shards, reads = [], []
    for r in range(world):
        a, b = plan.bounds(r)
        dgs = P.BvGraph(s, P.CreateOptions(row_begin=a, row_end=b))
        shards.append((a, b, dgs))
        reads.append(torch.from_numpy(dgs.read_set().astype(np.int64)).cuda())
    masks = []
    for r in range(world):  # bit p of row k: shard p reads global row a_r + k
        a, b = plan.bounds(r)
        m = torch.zeros(b - a, dtype=torch.uint8, device="cuda")
        for p_ in range(world):
            if p_ == r:
                continue
            rs = reads[p_]
            rs = rs[(rs >= a) & (rs < b)] - a
            m[rs] |= 1 << p_
        masks.append(m)
    nan = float("nan")
    qb = [[torch.full((n,), nan, dtype=torch.float64, device="cuda") for _ in range(2)] for _ in range(world)]
    dst = [torch.tensor([qb[p_][par].data_ptr() for p_ in range(world)], dtype=torch.int64, device="cuda")
           for par in (0, 1)]
    p = torch.full((n,), 1.0 / n, dtype=torch.float64, device="cuda")
    q0 = torch.where(deg > 0, p / deg.clamp(min=1).double(), torch.zeros_like(p))
    for r in range(world):  # iteration 0: own rows and read set (what the halo all_to_all delivers)
        a, b = plan.bounds(r)
        qb[r][0][a:b] = q0[a:b]
        qb[r][0][reads[r]] = q0[reads[r]]
    dmass = float(p[deg == 0].sum())
    for it in range(1, 21):
        cur, nxt = (it - 1) % 2, it % 2
        p_next = torch.empty_like(p)
        tot = torch.zeros(2, dtype=torch.float64, device="cuda")
        for r, (a, b, dgs) in enumerate(shards):
            part = torch.zeros(2, dtype=torch.float64, device="cuda")
            dgs.pagerank_step(qb[r][cur], deg[a:b], 0.15, dmass, "uniform", p[a:b], p_next[a:b], qb[r][nxt][a:b],
                              part, push_mask=masks[r], push_dst=dst[nxt])
            tot += part
        for r in range(world):  # the next iteration reads only pushed / own entries: poison the rest
            a, b = plan.bounds(r)
            keep = torch.zeros(n, dtype=torch.bool, device="cuda")
            keep[a:b] = True
            keep[reads[r]] = True
            qb[r][nxt].masked_fill_(~keep, nan)
            qb[r][cur].fill_(nan)
        p = p_next
        dmass = float(tot[0])
    want, _ = oracle_pr(g, iterations=20)
    assert rel(p.cpu().numpy(), want) <= 1e-12


@pytest.mark.parametrize("tol", [None, 1e-10])
def test_pagerank_start_vector(cuda, tol):
    """`start` (pagerank.hpp:86-102): the starting and restart distribution,
    validated as a probability vector -- against the oracle's pagerank with
    the same start, host and device buffers."""
    import torch

    g = make_graph(3, n=1 << 14)
    rng = np.random.default_rng(4)
    start = rng.random(g.n)
    start /= start.sum()
    dg = P.BvGraph(bv_of_transpose(g))
    og = O.Csr.from_arrays(g.n, g.row_offsets, g.columns)
    want, wit = O.pagerank_csr(og.transpose(), og.out_degrees(), 0.15, 40, l1_tolerance=tol, start=start)
    res = P.pagerank(P.BvGpuKernel(dg), g.out_degrees(), P.PageRankConfig(iterations=40, l1_tolerance=tol),
                     start=start)
    assert res.iterations_run == wit
    assert rel(res.ranks, want) <= 1e-12
    deg = torch.from_numpy(g.out_degrees().astype(np.int32)).cuda()
    p, it = dg.pagerank(deg, iterations=40, l1_tolerance=tol, start=torch.from_numpy(start).cuda())
    assert it == wit and rel(p.cpu().numpy(), want) <= 1e-12
    with pytest.raises(ValueError):
        P.pagerank(P.BvGpuKernel(dg), g.out_degrees(), P.PageRankConfig(iterations=5), start=start * 2)
    bad = start.copy()
    bad[0] = -bad[0]
    with pytest.raises(ValueError):
        P.pagerank(P.BvGpuKernel(dg), g.out_degrees(), P.PageRankConfig(iterations=5), start=bad)


def test_pagerank_equivalence_check(cuda):
    """cmv::pagerank_equivalence_check (pagerank.hpp:104-118): the CSR and the
    differential kernel give the same PageRank; the differential one needs
    fewer adds; compression stats as cmv::stats (ref_matrix.hpp:78-89)."""
    g = make_graph(3, n=1 << 15)
    eq = P.pagerank_equivalence_check(g, P.PageRankConfig(iterations=30), window=7)
    assert eq.iterations_run == 30
    assert eq.linf <= 1e-14
    assert eq.csr_adds == g.m and 0 < eq.ref_adds < eq.csr_adds
    c = eq.compression
    assert c.n == g.n and c.m == g.m and c.m_prime < c.m and abs(c.ratio - c.m / c.m_prime) < 1e-12
    assert 0 < c.rows_self_coded < g.n and 1 <= c.max_chain <= 3
    eq2 = P.pagerank_equivalence_check(g, P.PageRankConfig(iterations=200, l1_tolerance=1e-10), window=3)
    assert eq2.iterations_run < 200 and eq2.linf <= 1e-13


def test_pagerank_hub_rows_graph_capture(cuda):
    """PageRank on A^T of a power-law graph: hub rows (popular targets) spread
    over their block's chunks, in the device loop's captured CUDA graph;
    results match the oracle."""
    h = P.CsrGraph.social(1 << 15, seed=78)  # A^T: its hub rows are A's popular targets
    g = h.transpose()  # A
    dg = P.BvGraph(P.BvStream.encode(h, P.BvParams(max_ref=0)))
    assert dg.info()["bvf_max_K"] > 16
    p, it = dg.pagerank(g.out_degrees(), alpha=0.15, iterations=30)
    want, _ = oracle_pr(g, alpha=0.15, iterations=30, dangling="uniform")
    assert it == 30 and rel(p, want) <= 1e-12
