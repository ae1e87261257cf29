"""Row-sharded multi-GPU driver (one process per GPU, torch.distributed).

Sharding: rows are split into contiguous, block-aligned
shards; reference chains never leave a block, so every shard is
self-contained and the products need no data-path collective.  PageRank
(config 3) exchanges, per iteration, the new q = p/d of every shard
(all_gather into one n-vector laid out in row order) and two scalars
(dangling mass, L1 step) with all_reduce -- the only collectives.

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


def sharded_pagerank(step_fn: Callable, degrees_shard, n: int, plan: ShardPlan, rank: int, alpha: float = 0.15,
                     iterations: int = 10, l1_tolerance: Optional[float] = None, dangling: str = "uniform",
                     device=None, group=None):
    """Power iteration p_t = alpha/n + (1-alpha)(A^T q + D/n) over row shards.

    step_fn(q_full, alpha, dmass, p_prev_shard, p_next_shard, q_next_shard, partial) computes this shard's
    p_next / q_next and partial = [sum of p_next over dangling rows, L1 step] (device tensors).
    Returns (p_shard, iterations_run)."""
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
    dist.all_gather_into_tensor(q_pad, q_send, group=group)
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
        dist.all_gather_into_tensor(q_pad, q_next, group=group)
        dist.all_reduce(part, group=group)
        dmass = float(part[0].item())
        l1 = float(part[1].item())
        p, p_next = p_next, p
        if l1_tolerance is not None and l1 <= l1_tolerance:
            break
    return p, it


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
    buf = torch.zeros(plan.chunk, dtype=x_shard.dtype, device=x_shard.device)
    buf[: b - a] = x_shard
    full = torch.zeros(plan.world * plan.chunk, dtype=x_shard.dtype, device=x_shard.device)
    dist.all_gather_into_tensor(full, buf, group=group)
    return full[: plan.n].cpu().numpy() if rank == 0 else None
