"""Row-sharded multi-GPU driver (one process per GPU, torch.distributed).

Sharding: rows are split into contiguous, block-aligned
shards; reference chains never leave a block, so every shard is
self-contained and the products need no data-path collective.  PageRank
(config 3) exchanges, per iteration, the new q = p/d and two scalars
(dangling mass, L1 step, all_reduce).  The q exchange is either
  * full: all_gather of every shard's q into one n-vector (the correctness
    path), or
  * halo: each rank receives only the q entries its gather reads from other
    shards (`BvGraph.read_set()`: its blocks' x-windows -- mostly its own rows
    plus a slab at each edge -- and the rare out-of-window columns), with one
    all_to_all_single of precomputed index lists (`plan_halo`).  For the
    copy-model A^T of config 3 that is a small fraction of the full vector;
  * push: the halo exchange fused into the step kernel -- its epilogue stores
    each new q'_k straight into the q buffers of the peers that read row k
    (`plan_push` masks, NVLink peer memory from torch symmetric memory), so
    no separate collective moves q at all; the scalar all_reduce orders the
    iterations.

The per-shard compute is `BvGraph.pagerank_step` (one fused sm_100a kernel +
a reduction).  `step_fn` can be replaced for CPU testing of the exchange logic
(tests/test_distributed_cpu.py drives it with gloo and an oracle step).
"""
from __future__ import annotations

import dataclasses
from typing import Callable, Optional

import numpy as np


@dataclasses.dataclass
class ShardPlan:
    n: int
    world: int
    block_rows: int
    chunk: int  # rows per shard (multiple of block_rows); the last shard may be shorter

    def bounds(self, rank: int):
        a = min(self.n, rank * self.chunk)
        b = min(self.n, (rank + 1) * self.chunk)
        return a, b


def plan_shards(n: int, world: int, block_rows: int) -> ShardPlan:
    nblocks = (n + block_rows - 1) // block_rows
    per = (nblocks + world - 1) // world
    return ShardPlan(n=n, world=world, block_rows=block_rows, chunk=per * block_rows)


@dataclasses.dataclass
class HaloPlan:
    """Per-rank index lists of the halo exchange (see plan_halo)."""
    send_idx: object      # int64 tensor: local rows of my q to send, grouped by destination rank
    send_counts: list     # per destination rank
    recv_cols: object     # int64 tensor: global columns I receive, grouped by source rank
    recv_counts: list     # per source rank

    @property
    def recv_entries(self) -> int:
        return int(sum(self.recv_counts))


def plan_halo(read_set, plan: ShardPlan, rank: int, device=None, group=None) -> HaloPlan:
    """Exchange, once, which q entries each rank needs from each owner: the
    columns of `read_set` (sorted, unique) outside this rank's rows, grouped by
    owner shard.  Collective over the group."""
    import torch
    import torch.distributed as dist

    a, b = plan.bounds(rank)
    rs = np.asarray(read_set, dtype=np.int64)
    remote = rs[(rs < a) | (rs >= b)]
    owner = remote // plan.chunk  # sorted columns -> grouped by owner
    req_counts = np.bincount(owner, minlength=plan.world).astype(np.int64)
    req = torch.from_numpy(req_counts).to(device)
    got = torch.empty_like(req)
    dist.all_to_all_single(got, req, group=group)
    send_counts = [int(v) for v in got.cpu().tolist()]
    recv_counts = [int(v) for v in req_counts.tolist()]
    recv_cols = torch.from_numpy(remote).to(device)
    incoming = torch.empty(sum(send_counts), dtype=torch.int64, device=device)
    dist.all_to_all_single(incoming, recv_cols, output_split_sizes=send_counts, input_split_sizes=recv_counts,
                           group=group)
    return HaloPlan(send_idx=incoming - a, send_counts=send_counts, recv_cols=recv_cols, recv_counts=recv_counts)


def plan_push(halo: HaloPlan, plan: ShardPlan, rank: int, device=None):
    """Per shard row, the bit mask of the peer ranks that read it (from the
    halo plan's send lists): the fused push's destinations."""
    import torch

    a, b = plan.bounds(rank)
    mask = torch.zeros(b - a, dtype=torch.uint8, device=device)
    off = 0
    for p, c in enumerate(halo.send_counts):
        if c:
            idx = halo.send_idx[off:off + c].to(device)
            mask.index_put_((idx,), mask.index_select(0, idx) | (1 << p))
        off += c
    return mask


def sharded_pagerank(step_fn: Callable, degrees_shard, n: int, plan: ShardPlan, rank: int, alpha: float = 0.15,
                     iterations: int = 10, l1_tolerance: Optional[float] = None, dangling: str = "uniform",
                     device=None, group=None, halo: Optional[HaloPlan] = None):
    """Power iteration p_t = alpha/n + (1-alpha)(A^T q + D/n) over row shards.

    step_fn(q_full, alpha, dmass, p_prev_shard, p_next_shard, q_next_shard, partial) computes this shard's
    p_next / q_next and partial = [sum of p_next over dangling rows, L1 step] (device tensors).
    With `halo`, q_full holds correct values only at this rank's rows and its
    read set (all the step reads).  Returns (p_shard, iterations_run)."""
    import torch
    import torch.distributed as dist

    a, b = plan.bounds(rank)
    rows = b - a
    dt = torch.float64
    q_pad = torch.zeros(plan.world * plan.chunk, dtype=dt, device=device)
    deg = degrees_shard
    p = torch.full((rows,), 1.0 / n, dtype=dt, device=device)
    q_loc = torch.where(deg > 0, p / deg.clamp(min=1).to(dt), torch.zeros_like(p))
    q_send = torch.zeros(plan.chunk, dtype=dt, device=device)
    q_send[:rows] = q_loc
    if halo is not None:
        recv = torch.empty(halo.recv_entries, dtype=dt, device=device)

    def exchange(q_shard):
        if halo is None:
            dist.all_gather_into_tensor(q_pad, q_shard, group=group)
            return
        q_pad[a:b] = q_shard[:rows]
        send = q_shard.index_select(0, halo.send_idx)
        dist.all_to_all_single(recv, send, output_split_sizes=halo.recv_counts, input_split_sizes=halo.send_counts,
                               group=group)
        q_pad.index_copy_(0, halo.recv_cols, recv)

    exchange(q_send)
    part = torch.zeros(2, dtype=dt, device=device)
    part[0] = p[deg == 0].sum()
    dist.all_reduce(part, group=group)
    dmass = float(part[0].item())
    p_next = torch.empty_like(p)
    q_next = torch.empty(plan.chunk, dtype=dt, device=device)
    it = 0
    for it in range(1, iterations + 1):
        q_next.zero_()
        step_fn(q_pad[:n], alpha, dmass, p if l1_tolerance is not None else None, p_next, q_next[:rows], part)
        exchange(q_next)
        dist.all_reduce(part, group=group)
        dmass = float(part[0].item())
        l1 = float(part[1].item())
        p, p_next = p_next, p
        if l1_tolerance is not None and l1 <= l1_tolerance:
            break
    return p, it


def sharded_pagerank_dev(step_fn: Callable, degrees_shard, n: int, plan: ShardPlan, rank: int, alpha: float = 0.15,
                        iterations: int = 10, l1_tolerance: Optional[float] = None, dangling: str = "uniform",
                        device=None, group=None, halo: Optional[HaloPlan] = None, push=None):
    """sharded_pagerank with every per-iteration scalar kept on the device:
    step_fn(q_full, alpha, dmass_dev, p_prev, p_next, q_next, part_out) reads
    the dangling mass from dmass_dev[0] (the previous step's all-reduced
    partial sums; cmvg_pagerank_step_dev), so an iteration is step ->
    exchange -> all_reduce queued on the stream with no host round trip.  With
    l1_tolerance the L1 step is read back every iteration (the stop rule of
    pagerank.hpp:86-91 needs it); without it the loop never synchronises.
    `push` (a PushExchange) fuses the q exchange into the step kernel.
    Returns (p_shard, iterations_run)."""
    import torch
    import torch.distributed as dist

    a, b = plan.bounds(rank)
    rows = b - a
    dt = torch.float64
    deg = degrees_shard
    single = plan.world == 1 and not dist.is_initialized()  # one process: no collectives at all

    def all_reduce(t):
        if not single:
            dist.all_reduce(t, group=group)

    p = torch.full((rows,), 1.0 / n, dtype=dt, device=device)
    q_loc = torch.where(deg > 0, p / deg.clamp(min=1).to(dt), torch.zeros_like(p))
    part = [torch.zeros(2, dtype=dt, device=device), torch.zeros(2, dtype=dt, device=device)]
    part[0][0] = p[deg == 0].sum()
    all_reduce(part[0])
    p_next = torch.empty_like(p)
    if push is not None:
        q_bufs = push.qb
        push.prime(q_loc)
    else:
        # two full-length q vectors: iteration t reads buffer (t - 1) % 2 and the
        # step writes its own rows of buffer t % 2 in place, so no copy of the
        # shard's rows is made (at 1 GPU the loop is the step kernel alone)
        q_bufs = [torch.zeros(plan.world * plan.chunk, dtype=dt, device=device) for _ in range(2)]
        if halo is not None:
            recv = torch.empty(halo.recv_entries, dtype=dt, device=device)
        elif not single:
            q_send = torch.zeros(plan.chunk, dtype=dt, device=device)

        def exchange(qb):  # this shard's rows are in qb[a:b]
            if single:
                return
            if halo is None:
                q_send[:rows] = qb[a:b]
                dist.all_gather_into_tensor(qb, q_send, group=group)
                return
            dist.all_to_all_single(recv, qb[a:b].index_select(0, halo.send_idx), output_split_sizes=halo.recv_counts,
                                   input_split_sizes=halo.send_counts, group=group)
            qb.index_copy_(0, halo.recv_cols, recv)

        q_bufs[0][a:b] = q_loc
        exchange(q_bufs[0])
    it = 0
    for it in range(1, iterations + 1):
        prev, cur = part[(it - 1) % 2], part[it % 2]
        p_prev = p if l1_tolerance is not None else None
        c, nx = (it - 1) % 2, it % 2
        if push is not None:
            step_fn(q_bufs[c], alpha, prev, p_prev, p_next, q_bufs[nx][a:b], cur, push=push, parity=nx)
        else:
            step_fn(q_bufs[c][:n], alpha, prev, p_prev, p_next, q_bufs[nx][a:b], cur)
            exchange(q_bufs[nx])
        all_reduce(cur)
        p, p_next = p_next, p
        if l1_tolerance is not None and float(cur[1].item()) <= l1_tolerance:
            break
    return p, it


class PushExchange:
    """State of the fused exchange (world <= 8): two q buffers per rank in
    torch symmetric memory (peer-mapped over NVLink), the peer pointer tables
    for each parity and this shard's push masks.  Build once, run many."""

    def __init__(self, n: int, plan: ShardPlan, rank: int, halo: HaloPlan, device=None, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        if plan.world > 8:
            raise ValueError("the fused push addresses at most 8 peers")
        self.n, self.plan, self.rank, self.halo, self.device, self.group = n, plan, rank, halo, device, group
        self.buf = symm_mem.empty(2 * n, dtype=torch.float64, device=device)
        self.buf.zero_()
        hdl = symm_mem.rendezvous(self.buf, (group or dist.group.WORLD).group_name)
        ptrs = [int(hdl.buffer_ptrs[p]) for p in range(plan.world)]
        self.dst = [torch.tensor([ptrs[p] + par * n * 8 for p in range(plan.world)], dtype=torch.int64,
                                 device=device) for par in (0, 1)]
        self.qb = [self.buf[:n], self.buf[n:]]
        self.mask = plan_push(halo, plan, rank, device)
        self.recv = torch.empty(halo.recv_entries, dtype=torch.float64, device=device)

    def prime(self, q_shard):
        """Iteration 0's q: own rows into buffer 0, the halo by one all_to_all
        (every later one is pushed by the step kernel)."""
        import torch.distributed as dist

        a, b = self.plan.bounds(self.rank)
        q0 = self.qb[0]
        q0[a:b] = q_shard
        dist.all_to_all_single(self.recv, q_shard.index_select(0, self.halo.send_idx),
                               output_split_sizes=self.halo.recv_counts, input_split_sizes=self.halo.send_counts,
                               group=self.group)
        q0.index_copy_(0, self.halo.recv_cols, self.recv)

    def run(self, graph, degrees_shard, alpha: float = 0.15, iterations: int = 10,
            l1_tolerance: Optional[float] = None, dangling: str = "uniform"):
        """sharded_pagerank with the exchange fused into the step kernel:
        iteration t reads buffer t % 2; the kernel writes its rows of buffer
        (t+1) % 2 locally and into every peer that reads them
        (cmvg_pagerank_step_push).  The scalar all_reduce after each step
        orders it before any peer's next step, so two buffers suffice.
        Returns (p_shard, iterations_run)."""
        import torch
        import torch.distributed as dist

        n, plan, halo, dev, group = self.n, self.plan, self.halo, self.device, self.group
        a, b = plan.bounds(self.rank)
        dt = torch.float64
        deg = degrees_shard
        p = torch.full((b - a,), 1.0 / n, dtype=dt, device=dev)
        q0 = self.qb[0]
        q0[a:b] = torch.where(deg > 0, p / deg.clamp(min=1).to(dt), torch.zeros_like(p))
        # iteration 0's halo: one all_to_all (every later one is pushed by the kernel)
        dist.all_to_all_single(self.recv, q0[a:b].index_select(0, halo.send_idx),
                               output_split_sizes=halo.recv_counts, input_split_sizes=halo.send_counts, group=group)
        q0.index_copy_(0, halo.recv_cols, self.recv)
        part = torch.zeros(2, dtype=dt, device=dev)
        part[0] = p[deg == 0].sum()
        dist.all_reduce(part, group=group)
        dmass = float(part[0].item())
        p_next = torch.empty_like(p)
        it = 0
        for it in range(1, iterations + 1):
            cur, nxt = (it - 1) % 2, it % 2
            graph.pagerank_step(self.qb[cur], deg, alpha, dmass, dangling, p if l1_tolerance is not None else None,
                                p_next, self.qb[nxt][a:b], part, push_mask=self.mask, push_dst=self.dst[nxt])
            dist.all_reduce(part, group=group)
            dmass = float(part[0].item())
            l1 = float(part[1].item())
            p, p_next = p_next, p
            if l1_tolerance is not None and l1 <= l1_tolerance:
                break
        return p, it


def gpu_step_fn_dev(graph, degrees_shard, dangling: str = "uniform"):
    """The production step for sharded_pagerank_dev: the dangling mass stays on
    the device (cmvg_pagerank_step_dev); with a PushExchange the q exchange is
    fused into the kernel."""

    def step(q_full, alpha, dmass_dev, p_prev, p_next, q_next, part, push=None, parity=0):
        if push is None:
            graph.pagerank_step_dev(q_full, degrees_shard, alpha, dmass_dev, dangling, p_prev, p_next, q_next, part)
        else:
            graph.pagerank_step_dev(q_full, degrees_shard, alpha, dmass_dev, dangling, p_prev, p_next, q_next, part,
                                    push_mask=push.mask, push_dst=push.dst[parity])

    return step


def gpu_step_fn(graph, degrees_shard, dangling: str = "uniform"):
    """The production step: one fused gather+update kernel on this rank's shard."""

    def step(q_full, alpha, dmass, p_prev, p_next, q_next, part):
        graph.pagerank_step(q_full, degrees_shard, alpha, dmass, dangling, p_prev, p_next, q_next, part)

    return step


def gather_to_rank0(x_shard, plan: ShardPlan, rank: int, group=None):
    """Collect a row-sharded vector on every rank (row order); returns numpy on rank 0."""
    import torch
    import torch.distributed as dist

    a, b = plan.bounds(rank)
    if plan.world == 1 and not dist.is_initialized():
        return x_shard[: plan.n].cpu().numpy()
    buf = torch.zeros(plan.chunk, dtype=x_shard.dtype, device=x_shard.device)
    buf[: b - a] = x_shard
    full = torch.zeros(plan.world * plan.chunk, dtype=x_shard.dtype, device=x_shard.device)
    dist.all_gather_into_tensor(full, buf, group=group)
    return full[: plan.n].cpu().numpy() if rank == 0 else None
