"""The multi-GPU path's host logic on CPU: world_size 2 with gloo, the sharded
PageRank driver (shard plan, all_gather of q, all_reduce of the dangling mass
and L1 step) run with an oracle step per shard, checked against the
single-process oracle PageRank (pagerank.hpp:100-102)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import pyoracle as O
from paper_1708_07271_b200.distributed import plan_halo, plan_shards, sharded_pagerank, sharded_pagerank_dev


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _graph(n, seed):
    rng = np.random.default_rng(seed)
    m = n * 6
    src = rng.integers(0, n, m)
    dst = np.clip(src + rng.integers(-40, 40, m), 0, n - 1)
    keep = rng.random(m) < 0.9
    edges = np.stack([src[keep], dst[keep]], 1)
    return O.Csr.build(edges, n)


def _worker(rank, world, port, n, block_rows, iters, tol, out, use_halo=False, dev_scalars=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = _graph(n, 5)
    at = g.transpose()
    deg = g.out_degrees()
    plan = plan_shards(n, world, block_rows)
    a, b = plan.bounds(rank)
    ro, co = at.row_offsets, at.cols

    def step(q_full, alpha, dmass, p_prev, p_next, q_next, part):
        # oracle restatement of one shard's fused step (CPU stand-in for the kernel)
        if torch.is_tensor(dmass):  # sharded_pagerank_dev: the all-reduced partials of the previous step
            dmass = float(dmass[0])
        qf = q_full.numpy()
        y = np.array([qf[co[ro[i]:ro[i + 1]]].sum() for i in range(a, b)])
        pn = alpha / n + (1 - alpha) * (y + dmass / n)
        d = deg[a:b]
        p_next.copy_(torch.from_numpy(pn))
        q_next.copy_(torch.from_numpy(np.where(d > 0, pn / np.maximum(d, 1), 0.0)))
        part[0] = float(pn[d == 0].sum())
        part[1] = float(np.abs(pn - p_prev.numpy()).sum()) if p_prev is not None else 0.0

    halo = None
    if use_halo:
        # the columns this shard's step reads (the GPU path gets them from BvGraph.read_set())
        rs = np.unique(co[ro[a]:ro[b]]).astype(np.uint32)
        halo = plan_halo(rs, plan, rank)
        assert halo.recv_entries < n  # strictly less than a full all_gather

    def poisoned_step(q_full, *args):
        if halo is not None:  # entries outside the read set and own rows must not be used
            keep = torch.zeros(n, dtype=torch.bool)
            keep[a:b] = True
            keep[torch.from_numpy(np.unique(co[ro[a]:ro[b]]).astype(np.int64))] = True
            q_full = torch.where(keep, q_full, torch.full_like(q_full, float("nan")))
        step(q_full, *args)

    driver = sharded_pagerank_dev if dev_scalars else sharded_pagerank
    p, it = driver(poisoned_step, torch.from_numpy(deg[a:b].astype(np.int64)), n, plan, rank, 0.15, iters, tol,
                   halo=halo)
    full = torch.zeros(plan.world * plan.chunk, dtype=torch.float64)
    buf = torch.zeros(plan.chunk, dtype=torch.float64)
    buf[: b - a] = p
    dist.all_gather_into_tensor(full, buf)
    if rank == 0:
        np.save(out, np.concatenate([full[:n].numpy(), [it]]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,block_rows,iters,tol,halo,dev", [(2, 5000, 1024, 30, None, False, False),
                                                                   (2, 3000, 1024, 200, 1e-9, False, False),
                                                                   (3, 4100, 512, 20, None, False, False),
                                                                   (2, 5000, 1024, 30, None, True, False),
                                                                   (3, 4100, 512, 40, 1e-9, True, False),
                                                                   (2, 5000, 1024, 30, None, True, True),
                                                                   (3, 4100, 512, 40, 1e-9, False, True),
                                                                   (2, 3000, 1024, 200, 1e-9, True, True)])
def test_sharded_pagerank_matches_oracle(tmp_path, world, n, block_rows, iters, tol, halo, dev):
    out = str(tmp_path / "p.npy")
    mp.spawn(_worker, args=(world, _free_port(), n, block_rows, iters, tol, out, halo, dev), nprocs=world, join=True)
    got = np.load(out)
    p, it = got[:n], int(got[n])
    g = _graph(n, 5)
    want, want_it = O.pagerank_csr(g.transpose(), g.out_degrees(), 0.15, iters, l1_tolerance=tol)
    assert it == want_it
    assert np.max(np.abs(p - want) / want) <= 1e-12
    assert abs(p.sum() - 1.0) <= 1e-10


def test_shard_plan_block_aligned():
    plan = plan_shards(10_000, 3, 1024)
    bounds = [plan.bounds(r) for r in range(3)]
    assert bounds[0][0] == 0 and bounds[-1][1] == 10_000
    for (a, b), (c, d) in zip(bounds, bounds[1:]):
        assert b == c and a % 1024 == 0
    assert plan.chunk % 1024 == 0


def _push_worker(rank, world, port, n, out):
    from paper_1708_07271_b200.distributed import plan_push

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = _graph(n, 5)
    at = g.transpose()
    plan = plan_shards(n, world, 512)
    a, b = plan.bounds(rank)
    ro, co = at.row_offsets, at.cols
    rs = np.unique(co[ro[a]:ro[b]]).astype(np.uint32)
    mask = plan_push(plan_halo(rs, plan, rank), plan, rank)
    full = [None] * world
    dist.all_gather_object(full, (rank, rs.tolist(), mask.numpy().tolist()))
    if rank == 0:
        import pickle

        pickle.dump(full, open(out, "wb"))
    dist.destroy_process_group()


def test_push_masks_match_read_sets(tmp_path):
    """plan_push: bit p of shard-row k is set exactly when rank p's read set
    holds that global row (and p is not the owner)."""
    import pickle

    world, n = 3, 4000
    out = str(tmp_path / "m.pkl")
    mp.spawn(_push_worker, args=(world, _free_port(), n, out), nprocs=world, join=True)
    full = sorted(pickle.load(open(out, "rb")))
    plan = plan_shards(n, world, 512)
    reads = [set(r) for _, r, _ in full]
    for rank, _, mask in full:
        a, b = plan.bounds(rank)
        assert len(mask) == b - a
        for k, m in enumerate(mask):
            want = sum(1 << p for p in range(world) if p != rank and (a + k) in reads[p])
            assert m == want, (rank, k, m, want)
