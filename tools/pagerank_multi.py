"""Sharded PageRank on config 3 (A^T of a copy model), one process per GPU.

    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \\
        --master-port 29511 tools/pagerank_multi.py [--n-log2 26] [--iters 50] [--exchange push|halo|full]

Each rank builds the BV stream of A^T (deterministic), owns a block-aligned
row shard (`plan_shards`), and runs the fused GPU step; the q exchange is the
kernel's own push into the peers' symmetric-memory buffers (default), the halo
all_to_all, or the full all_gather.  Rank 0 prints
one JSON line: iterations/s (device time, max over ranks), the halo volume,
and -- for n <= 2^22 -- parity against the CPU oracle.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-log2", type=int, default=26)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--exchange", choices=["push", "halo", "full"], default="push")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_1708_07271_b200 as P
    from paper_1708_07271_b200.distributed import (PushExchange, gather_to_rank0, gpu_step_fn_dev, plan_halo,
                                                   plan_shards, sharded_pagerank_dev)

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29511")
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    n = 1 << args.n_log2
    g = P.CsrGraph.copy_model(n, 24.0, 0.7, 0.8, seed=0x170807271 + 3)
    s = P.BvStream.encode(g.transpose(), P.BvParams())
    plan = plan_shards(n, world, 1024)
    a, b = plan.bounds(rank)
    t0 = time.time()
    dg = P.BvGraph(s, P.CreateOptions(device=local, row_begin=a, row_end=b))
    build_s = time.time() - t0
    deg_all = g.out_degrees()
    deg = torch.from_numpy(deg_all[a:b].astype(np.int32)).to(dev)
    halo = plan_halo(dg.read_set(), plan, rank, device=dev) if args.exchange != "full" else None
    step = gpu_step_fn_dev(dg, deg)  # every per-iteration scalar stays on the device
    push = PushExchange(n, plan, rank, halo, device=dev) if args.exchange == "push" else None

    def run(iters):
        if push is not None:
            return push.run(dg, deg, iterations=iters)
        return sharded_pagerank_dev(step, deg, n, plan, rank, iterations=iters, device=dev, halo=halo)
    run(2)  # warm-up
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    p, it = run(args.iters)
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    recv = torch.tensor([halo.recv_entries if halo else n - (b - a)], dtype=torch.float64, device=dev)
    dist.all_reduce(recv, op=dist.ReduceOp.MAX)
    full = gather_to_rank0(p, plan, rank)
    if rank == 0:
        out = {"workload": f"C3 PageRank n=2^{args.n_log2} m={g.m}", "n_gpus": world, "exchange": args.exchange,
               "iterations": it, "ms_per_iter": float(ms.item()) / it, "iter_per_s": it / float(ms.item()) * 1e3,
               "max_recv_entries_per_iter": int(recv.item()), "full_vector_entries": n, "build_s": build_s}
        if n <= (1 << 22):
            from oracle import pyoracle as O

            og = O.Csr.from_arrays(n, g.row_offsets, g.columns)
            want, _ = O.pagerank_csr(og.transpose(), og.out_degrees(), 0.15, it)
            out["max_rel_err"] = float(np.max(np.abs(full - want) / want))
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
