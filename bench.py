#!/usr/bin/env python
"""Headline benchmark: compressed A·x on B200 (BASELINE.json metric
"compressed A·x Gedges/s ... % HBM roofline ...").

Workload: BASELINE.json configs[1] (C2): synthetic copy-model graph,
n = 2^24, mean out-degree 20, BV w=7 R=3 Lmin=4 zeta_3, one y = A x^T in fp64
per step with x ~ U[0,1) resident in HBM.  Under torchrun the rows are sharded
over the ranks (block-aligned shards, x replicated, y sharded: strong scaling,
no data-path collective).  Beside it, a sharded PageRank leg (C3 generator,
q exchanged per iteration over NCCL, all scalars device resident).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Prints ONE JSON line (rank 0).  See DESIGN.md §Measurement for every field.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 0x170807271
L2_FLUSH_BYTES = 512 << 20  # > 126 MB L2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n-log2", type=int, default=24, help="rows = 2^n_log2 (C2: 24)")
    ap.add_argument("--degree", type=float, default=20.0)
    ap.add_argument("--dtype", choices=["f64", "f32"], default="f64")
    ap.add_argument("--form", choices=["gather", "scatter"], default="gather")
    ap.add_argument("--lanes", type=int, default=256)
    ap.add_argument("--block-rows", type=int, default=1024)
    ap.add_argument("--window", type=int, default=1536)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--no-csr", action="store_true", help="skip the uncompressed GPU CSR comparison")
    ap.add_argument("--secondary", action="store_true", help="also time the f32 / scatter variants (stderr)")
    ap.add_argument("--cpu-sample-seconds", type=float, default=20.0)
    ap.add_argument("--no-pagerank", action="store_true", help="skip the sharded PageRank leg")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle parity checks (profiling runs)")
    ap.add_argument("--pr-log2", type=int, default=0,
                    help="PageRank leg: n = 2^pr_log2 (default: the full C3 size 26 at 1 GPU, 24 under torchrun, "
                         "where every rank generates the whole graph)")
    ap.add_argument("--pr-iters", type=int, default=50, help="PageRank leg iterations (C3: 50)")
    ap.add_argument("--c4-log2", type=int, default=-1,
                    help="C4 leg (social graph, R = unbounded, y = A x^T in fp32, rows sharded): n = 2^c4_log2 "
                         "(BASELINE.json configs[3]: 25); 0 skips it; default 25 at 1-2 GPUs, skipped at more "
                         "(every rank generates and encodes the whole 1e9-edge graph on the shared host cores)")
    ap.add_argument("--pr-exchange", choices=["halo", "push"], default="halo",
                    help="PageRank leg at N > 1: halo all_to_all (NCCL) or the fused push of q' into the peers' "
                         "symmetric-memory buffers from the step kernel")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index: int, enabled: bool):
        self.proc = None
        self.path = os.path.join("/tmp", f"cmvg_clocks_{os.getpid()}.csv")
        if not enabled:
            return
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = max(smax, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


def workload_label(args) -> str:
    """The workload string of BOTH arms (same_config is checked on it)."""
    return (f"C2 copy-model n=2^{args.n_log2} deg{args.degree:g} y=A·x^T ({args.form}) {args.dtype} "
            f"(BASELINE.json configs[1])")


def make_workload(args, rank):
    import paper_1708_07271_b200 as P

    n = 1 << args.n_log2
    t0 = time.time()
    g = P.CsrGraph.copy_model(n, args.degree, 0.7, 0.8, seed=SEED + 2)
    t1 = time.time()
    s = P.BvStream.encode(g, P.BvParams(window=7, max_ref=3, min_interval=4, zeta_k=3, segment_rows=1024))
    t2 = time.time()
    log(f"[rank {rank}] generated n={g.n} m={g.m} in {t1 - t0:.1f}s, BV-encoded in {t2 - t1:.1f}s "
        f"({s.stats()['stream_bits'] / g.m:.3f} bits/edge)")
    return g, s


def x_uniform(n, seed, dtype):
    rng = np.random.default_rng(seed)
    x = (rng.integers(0, 2**64, size=n, dtype=np.uint64) >> np.uint64(11)).astype(np.float64) * 2.0**-53
    return x if dtype == "f64" else x.astype(np.float32)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference_throughput(n, ro, co, m, x64, steps, warmup, budget_s, threads=None):
    """The reference's own path restated (oracle): matvec_ref_into on
    compress(g, 7), sequential per product, run as `threads`
    concurrent independent products (SPEC.md:228 allows that) on the host
    cores.  Returns (edges/s, sample description, cores, per-step values)."""
    from oracle import pyoracle as O

    threads = threads or O.threads()
    t0 = time.time()
    og = O.Csr.from_arrays(n, ro, co)
    rm = O.RefMatrix.compress(og, 7, threads)
    tc = time.time() - t0
    log(f"[cpu] compress(g,7) with {threads} threads took {tc:.1f}s")
    vals = []
    t_start = time.time()
    for k in range(warmup + steps):
        sec = rm.matvec_concurrent(x64, threads)
        if k >= warmup:
            vals.append(threads * m / sec)
        if time.time() - t_start > budget_s and len(vals) >= 1:
            break
    sample = (f"{len(vals)} timed rounds of {threads} concurrent full matvec_ref products "
              f"(n={n}, m={m}) on compress(g,7); compress took {tc:.1f}s")
    return float(np.median(vals)), sample, threads, vals


def cpu_csr_legs(n, ro, co, m, x64, reps=3):
    """the reference's matvec_csr_into (csr.hpp:53-55), one
    full product on 1 core and on all cores (row-parallel, partition-
    independent); median of `reps`, edges/s."""
    from oracle import pyoracle as O

    out = {}
    for th in (1, O.threads()):
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            O.matvec_csr_raw(n, ro, co, x64, th)
            ts.append(time.perf_counter() - t0)
        out[f"matvec_csr_{th}t"] = {"gedges_s": m / float(np.median(ts)) / 1e9, "ms": float(np.median(ts)) * 1e3,
                                    "threads": th}
    return out


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU reference
    from oracle import pyoracle as O  # generator compiled alone (libcmv_gen.so): no product library here

    n = 1 << args.n_log2
    n, ro, co = O.generate_copy_model(n, args.degree, 0.7, 0.8, seed=SEED + 2)
    m = int(ro[-1])
    x64 = x_uniform(n, 11, "f64")
    v, sample, cores, _ = cpu_reference_throughput(n, ro, co, m, x64, args.steps, args.warmup, budget_s=1e9)
    gv = v / 1e9
    out = {
        "metric": "compressed A·x Gedges/s", "value": gv, "unit": "Gedges/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": m / v * 1e3 * cores,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "impl": "reference",
        "config": {"workload": workload_label(args), "n": n, "m": m,
                   "reference_format": "compress(g,7) A' (ref_matrix.hpp:69)"},
        "cpu_baseline": {"value": gv, "unit": "Gedges/s", "cores": cores, "kind": "port", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": gv, "unit": "Gedges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def timed_events(fn, steps, flush, stream):
    """CUDA events around each of `steps` launches of fn on `stream`, L2
    flushed before each (outside the events); returns ms per launch."""
    import torch

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in evs:
        flush.zero_()
        a.record(stream)
        fn()
        b.record(stream)
    torch.cuda.synchronize()
    return np.array([a.elapsed_time(b) for a, b in evs])


def max_over_ranks(v, dev, world):
    import torch
    import torch.distributed as dist

    if world == 1:
        return float(v)
    t = torch.tensor([float(v)], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def pagerank_leg(args, dev, rank, world, plan_fn, flush):
    """PageRank on BV(A^T) of the C3 generator (BASELINE.json configs[2]:
    copy model, mean degree 24, alpha 0.15, uniform dangling) at n = 2^pr_log2,
    rows sharded over the ranks; q exchanged per iteration by the halo
    all_to_all (NCCL) with all scalars device resident
    (distributed.sharded_pagerank_dev).  Iterations timed by CUDA events, max
    over ranks.  Informational beside the headline (full C3 is n = 2^26:
    --pr-log2 26)."""
    import torch
    import torch.distributed as dist

    import paper_1708_07271_b200 as P
    from paper_1708_07271_b200 import distributed as D

    n = 1 << args.pr_log2
    t0 = time.time()
    g = P.CsrGraph.copy_model(n, 24.0, 0.7, 0.8, seed=SEED + 3)  # C3 generator (tests/helpers.py CONFIGS[3])
    at = g.transpose()
    s = P.BvStream.encode(at, P.BvParams(window=7, max_ref=3, min_interval=4, zeta_k=3, segment_rows=1024))
    plan = D.plan_shards(n, world, args.block_rows)
    a, b = plan.bounds(rank)
    dg = P.BvGraph(s, P.CreateOptions(device=dev.index, block_rows=args.block_rows, window=args.window,
                                      row_begin=a, row_end=b))
    log(f"[rank {rank}] pagerank graph n={n} m={g.m} ready in {time.time() - t0:.1f}s")
    deg_all = g.out_degrees().astype(np.int32)
    deg = torch.from_numpy(deg_all[a:b]).to(dev)
    step = D.gpu_step_fn_dev(dg, deg)
    halo = None
    if world > 1:
        halo = D.plan_halo(dg.read_set(), plan, rank, device=dev)
    iters = args.pr_iters

    push = None
    if world > 1 and args.pr_exchange == "push":
        push = D.PushExchange(n, plan, rank, halo, device=dev)

    def run(k):
        if push is not None:
            return push.run(dg, deg, alpha=0.15, iterations=k)
        return D.sharded_pagerank_dev(step, deg, n, plan, rank, 0.15, k, None, device=dev, halo=halo)

    run(3)  # warm-up (attributes, NCCL)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    flush.zero_()
    torch.cuda.synchronize()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record()
    p, it = run(iters)
    eb.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(ea.elapsed_time(eb), dev, world)
    out = {"iter_s": iters / (ms * 1e-3), "ms_per_iter": ms / iters, "iterations": iters, "n": n, "m": g.m,
           "exchange": ("fused push of q' into the peers' symmetric memory from the step kernel" if push is not None
                        else "halo all_to_all (NCCL), scalars device resident") if world > 1 else "none (1 GPU)",
           "what": f"PageRank alpha=0.15 kUniform on BV(A^T), C3 generator at n=2^{args.pr_log2}, rows sharded x{world}; "
                   "timed region = the whole iteration loop incl. initialisation (CUDA events, max over ranks)"}
    full = D.gather_to_rank0(p, plan, rank)
    if rank == 0 and not args.no_parity:
        from oracle import pyoracle as O
        want, _ = O.pagerank_csr(O.Csr.from_arrays(n, at.row_offsets, at.columns), deg_all.astype(np.uint32), 0.15,
                                 iters, nthreads=O.threads())
        out["parity_max_rel_err"] = float(np.max(np.abs(full - want) / want))
        out["sum_p_minus_1"] = float(abs(full.sum() - 1.0))
    del dg
    return out


def c4_leg(args, dev, rank, world, flush):
    """C4 (BASELINE.json configs[3]): the social generator (Zipf 2.1 out-degrees,
    80% of successors in the node's 4096-node community), BV w=7 with
    unbounded reference chains, one y = A x^T in fp32 per step; rows sharded
    over the ranks (block-aligned, x replicated, y sharded, no collective:
    strong scaling), a community-sized x-window (3968 entries).  Steps timed by
    CUDA events with the L2 flushed before each, max over ranks; parity on
    rank 0 against the oracle's matvec_csr of the fp32 x in fp64 (1e-5)."""
    import torch

    import paper_1708_07271_b200 as P
    from paper_1708_07271_b200 import distributed as D

    n = 1 << args.c4_log2
    t0 = time.time()
    g = P.CsrGraph.social(n, seed=SEED + 4)
    s = P.BvStream.encode(g, P.BvParams(window=7, max_ref=0, min_interval=4, zeta_k=3, segment_rows=1024))
    plan = D.plan_shards(n, world, args.block_rows)
    a, b = plan.bounds(rank)
    dg = P.BvGraph(s, P.CreateOptions(device=dev.index, block_rows=args.block_rows, window=3968,
                                      row_begin=a, row_end=b))
    info = dg.info()
    log(f"[rank {rank}] C4 graph n={n} m={g.m} ({s.stats()['stream_bits'] / g.m:.2f} bits/edge) rows [{a},{b}) "
        f"ready in {time.time() - t0:.1f}s, depth {info['max_depth']}")
    x64 = x_uniform(n, SEED + 40, "f64")
    x = torch.from_numpy(x64.astype(np.float32)).to(dev)
    y = torch.empty(b - a, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    def step():
        dg.matvec(x, y, stream=stream.cuda_stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    times = timed_events(step, args.steps, flush, stream)
    ms = max_over_ranks(float(times.mean()), dev, world)
    out = {"gedges_s": g.m / (ms * 1e-3) / 1e9, "ms": ms, "n": n, "m": g.m, "shard_rows_rank0": [a, b],
           "bits_per_edge": s.stats()["stream_bits"] / g.m, "max_depth": info["max_depth"],
           "window": 3968, "window_coverage": info.get("window_coverage"),
           "escape_terms_rank0": info.get("bvf_esc_terms"),
           "what": f"C4 social graph (R = unbounded) y = A x^T fp32 at n=2^{args.c4_log2}, rows sharded x{world} "
                   "(x replicated, y sharded, no collective); escape pre-gather + gather per step, CUDA events, "
                   "L2 flushed before each step, max over ranks"}
    if rank == 0 and world == 1 and not args.no_parity:
        from oracle import pyoracle as O
        want = O.matvec_csr_raw(n, g.row_offsets, g.columns, x64.astype(np.float32).astype(np.float64), O.threads())
        got = y.double().cpu().numpy()
        den = np.abs(want)
        err = np.abs(got - want)
        out["parity_max_rel_err"] = float(np.max(np.where(den > 0, err / np.where(den > 0, den, 1.0), err)))
    del dg
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1708_07271_b200 as P
    from paper_1708_07271_b200 import distributed as D

    rank, world, local = dist_env()
    if not args.pr_log2:  # the full C3 size at 1 GPU; under torchrun every rank generates the whole graph
        args.pr_log2 = 26 if world == 1 else 24
    if args.c4_log2 < 0:
        args.c4_log2 = 25 if world <= 2 else 0
    if world != args.gpus:
        args.gpus = world
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    g, s = make_workload(args, rank)
    # rows sharded over the ranks (block aligned; strong scaling: the job is
    # one product over the whole graph; x replicated, y stays sharded)
    plan = D.plan_shards(g.n, world, args.block_rows)
    a, b = plan.bounds(rank)
    opts = P.CreateOptions(device=local, block_rows=args.block_rows, lanes=args.lanes, window=args.window,
                           row_begin=a, row_end=b)
    t0 = time.time()
    dg = P.BvGraph(s, opts)
    info = dg.info()
    log(f"[rank {rank}] device handle rows [{a},{b}) built in {time.time() - t0:.1f}s: "
        f"BV-F {info['bvf_stream_bytes'] / 1e6:.1f} MB, terms {info['bvf_terms']}, pad {info['bvf_pad_terms']}")
    seg = s.segment_offsets()
    S = int(s.stats()["stream_bits"])
    seg_rows = 1024
    S_shard = int(seg[min(len(seg) - 1, (b + seg_rows - 1) // seg_rows)] - seg[a // seg_rows])
    xsz = 8 if args.dtype == "f64" else 4
    xh = x_uniform(g.n, 11, args.dtype)
    x = torch.from_numpy(xh).to(dev)
    y = torch.empty(b - a, dtype=x.dtype, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        dg.matvec(x, y, form=args.form, stream=stream.cuda_stream)

    sampler = ClockSampler(local, enabled=not args.no_clocks)
    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize(dev)

    def keep_busy(seconds):  # same launches, untimed: lets nvidia-smi sample clocks under this load
        if args.no_clocks:
            return
        t_end = time.time() + seconds
        while time.time() < t_end:
            for _ in range(8):
                flush.zero_()
                step()
            torch.cuda.synchronize(dev)

    keep_busy(0.6)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    times = timed_events(step, args.steps, flush, stream)
    if world > 1:
        dist.barrier()
    keep_busy(0.4)
    clocks = sampler.stop()
    if clocks is not None:
        clocks["how"] = "nvidia-smi -lms 50 across warm-up, the timed steps and surrounding identical untimed launches"
    t_rank = float(times.mean())
    t_mean = max_over_ranks(t_rank, dev, world)
    value = g.m / (t_mean * 1e-3) / 1e9  # the whole graph's edges per step (strong scaling)

    # roofline of the (only) kernel on rank 0: algorithmic bytes of its shard
    alg_bytes = math.ceil(S_shard / 8) + (b - a) * xsz + (b - a) * xsz
    peak, peak_src = measured_peak()
    achieved = alg_bytes / (t_rank * 1e-3) / 1e9
    traffic = None  # dram bytes per launch of this kernel from the committed ncu --set full capture
    prof = os.path.join(ROOT, "profiles", "ncu_gather_summary.json")
    if os.path.exists(prof) and world == 1:
        try:
            pj = json.load(open(prof))
            key = f"{args.form}_{args.dtype}_n{args.n_log2}_w{args.window}"
            if key in pj:
                traffic = pj[key]["dram_bytes_per_launch"]
        except Exception:
            traffic = None

    # e2e through the C-ABI host-pointer path (H2D + kernel + D2H each step):
    # pinned buffers (the pipelined path) and, at 1 GPU, ordinary pageable
    # numpy arrays (what MatvecKernel::multiply receives)
    e2e = None
    e2e_pageable = None
    if not args.no_e2e:
        def host_run(xin, yout):
            e_times = []
            for _ in range(max(1, args.warmup // 2)):
                dg.matvec(xin, yout, form=args.form)
            torch.cuda.synchronize(dev)
            if world > 1:
                dist.barrier()
            for _ in range(args.steps):
                flush.zero_()
                torch.cuda.synchronize(dev)
                t0 = time.perf_counter()
                dg.matvec(xin, yout, form=args.form)  # synchronous: copies + kernel
                e_times.append(time.perf_counter() - t0)
            return max_over_ranks(float(np.mean(e_times)), dev, world)

        xpin = torch.from_numpy(xh).pin_memory().numpy()
        ypin = torch.empty(b - a, dtype=x.dtype).pin_memory().numpy()
        te = host_run(xpin, ypin)
        e2e = {"value": g.m / te / 1e9, "unit": "Gedges/s", "h2d_bytes_per_step": g.n * xsz * world,
               "d2h_bytes_per_step": g.n * xsz, "ms_per_step": te * 1e3,
               "how": "cmvg_matvec_* with HOST pointers (pinned; x to every rank, y shard back); wall clock around "
                      "the synchronous call, max over ranks"}
        if world == 1:
            xpg = np.array(xh, copy=True)
            ypg = np.empty(b - a, dtype=xh.dtype)
            tp = host_run(xpg, ypg)
            e2e_pageable = {"value": g.m / tp / 1e9, "unit": "Gedges/s", "ms_per_step": tp * 1e3,
                            "how": "the same call with ordinary (pageable) numpy buffers"}

    # correctness spot check against the oracle's matvec_csr (rank 0's rows, outside timing)
    parity = None
    want = None
    if rank == 0 and not args.no_parity:
        from oracle import pyoracle as O
        want = O.matvec_csr_raw(g.n, g.row_offsets, g.columns, np.ascontiguousarray(xh, dtype=np.float64),
                                O.threads())
        got = y.double().cpu().numpy() if args.form == "gather" else None
        if got is not None:
            w = want[a:b]
            nz = w != 0
            parity = float(np.max(np.abs(got[nz] - w[nz]) / np.abs(w[nz])))
            parity = {"max_rel_err": parity, "zero_rows_exact": bool(np.all(got[~nz] == 0))}["max_rel_err"] if np.all(got[~nz] == 0) else float("inf")

    # uncompressed comparison point at equal hardware: the reference's
    # matvec_csr as a hand-written CSR kernel on the same GPU (PAPER.md:217's
    # S = t/t'), same x, same L2 flush; rank 0 at 1 GPU, outside the timed region
    csr_base = None
    if rank == 0 and world == 1 and args.form == "gather" and args.dtype == "f64" and not args.no_csr:
        ro = torch.from_numpy(g.row_offsets.astype(np.int64)).to(dev)
        co = torch.from_numpy(g.columns.view(np.int32)).to(dev)
        yc = torch.empty_like(x)
        for _ in range(args.warmup):
            flush.zero_()
            P.csr_matvec_device(ro, co, x, yc, stream=stream.cuda_stream)
        tc = float(timed_events(lambda: P.csr_matvec_device(ro, co, x, yc, stream=stream.cuda_stream), args.steps,
                                flush, stream).mean())
        csr_bytes = 4 * g.m + 8 * (g.n + 1) + 16 * g.n
        csr_base = {"ms": tc, "gedges_s": g.m / (tc * 1e-3) / 1e9, "bv_speedup": tc / t_rank,
                    "bytes_per_launch": csr_bytes, "gbs": csr_bytes / (tc * 1e-3) / 1e9,
                    "roofline_ms": csr_bytes / (peak * 1e9) * 1e3,
                    "bv_speedup_vs_csr_roofline": csr_bytes / (peak * 1e9) / (t_rank * 1e-3),
                    "what": "hand-written GPU CSR product (u64 row offsets, u32 columns, fp64; matvec_csr, "
                            "csr.hpp:48-55) on the same B200: bv_speedup = t_csr / t_compressed, the paper's "
                            "S = t/t' (PAPER.md:217) at equal hardware; roofline_ms = the CSR bytes at peak HBM "
                            "bandwidth (an ideal CSR kernel), bv_speedup_vs_csr_roofline = roofline_ms / t_compressed"}
        if want is not None:
            wc = yc.cpu().numpy()
            nz = want != 0
            csr_base["parity_max_rel_err"] = float(np.max(np.abs(wc[nz] - want[nz]) / np.abs(want[nz])))
        del ro, co, yc

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        x64 = np.ascontiguousarray(xh, dtype=np.float64)
        v, sample, cores, _ = cpu_reference_throughput(g.n, g.row_offsets, g.columns, g.m, x64, steps=3, warmup=1,
                                                       budget_s=args.cpu_sample_seconds)
        cpu = {"value": v / 1e9, "unit": "Gedges/s", "cores": cores, "kind": "port", "sample": sample,
               "cpu_model": cpu_model(), "csr_legs": cpu_csr_legs(g.n, g.row_offsets, g.columns, g.m, x64)}
        # SURVEY.md §8d (iii), informational: the product on the north-star format on one core --
        # the host codec's BV decode of the whole stream, then matvec_csr on one thread
        t0 = time.perf_counter()
        gd = s.decode_host()
        t_dec = time.perf_counter() - t0
        t_csr = cpu["csr_legs"]["matvec_csr_1t"]["ms"] * 1e-3
        cpu["bv_decode_product_1t"] = {"gedges_s": g.m / (t_dec + t_csr) / 1e9, "decode_s": t_dec,
                                       "product_s": t_csr, "threads": 1,
                                       "decoded_bit_exact": bool(np.array_equal(gd.columns, g.columns))}
        del gd

    pagerank = None
    del dg
    if not args.no_pagerank:
        pagerank = pagerank_leg(args, dev, rank, world, D.plan_shards, flush)
    c4 = None
    if args.c4_log2:
        c4 = c4_leg(args, dev, rank, world, flush)

    secondary = {}
    if args.secondary and rank == 0 and world == 1:
        secondary = run_secondary(args, g, s, dev)

    if rank == 0:
        out = {
            "metric": "compressed A·x Gedges/s", "value": value, "unit": "Gedges/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_mean, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": {
                "workload": workload_label(args),
                "n": g.n, "m": g.m, "bv": "w=7 R=3 Lmin=4 zeta3 segment=1024",
                "S_bits": S, "bits_per_edge": S / g.m,
                "device_layout": "BV-F (flat term stream)",
                "device_layout_bytes": info["bvf_stream_bytes"] + info["bvd_block_table_bytes"],
                "block_rows": args.block_rows, "window": args.window,
                "l2": "flushed (512 MiB write) before every timed launch",
                "parallelism": f"row shards x{world} (block aligned, x replicated, y sharded, no collective)",
                "shard_rows_rank0": [a, b],
            },
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "alg_bytes_per_launch": alg_bytes,
                         "alg_bytes_formula": "ceil(S_shard/8) + rows*sizeof(x) + rows*sizeof(y) (rank 0's shard; "
                                              "= ceil(S/8) + 2n*sizeof at 1 GPU)"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_pageable": e2e_pageable,
            # the gather kernel per step, plus the escape pre-gather when the shard has escape terms
            "gpu_launches": args.steps * (2 if info.get("bvf_esc_terms", 0) else 1),
            "clocks": clocks,
            "parity_max_rel_err_vs_matvec_csr": parity,
            "csr_baseline": csr_base,
            "kernel_ms": {"mean": t_rank, "median": float(np.median(times)), "min": float(times.min()),
                          "max": float(times.max())},
            "pagerank": pagerank,
            "c4": c4,
        }
        if secondary:
            out["secondary"] = secondary
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_secondary(args, g, s, dev):
    """Other variants on the same graph (reported, not the headline)."""
    import torch

    import paper_1708_07271_b200 as P

    res = {}
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    for dtype in ("f64", "f32"):
        for form in ("gather", "scatter"):
            try:
                dg = P.BvGraph(s, P.CreateOptions(device=dev.index, lanes=args.lanes, block_rows=args.block_rows,
                                                  window=args.window))
                xh = x_uniform(g.n, 11, dtype)
                x = torch.from_numpy(xh).to(dev)
                y = torch.empty(g.n, dtype=x.dtype, device=dev)
                for _ in range(3):
                    dg.matvec(x, y, form=form)
                ts = []
                for _ in range(10):
                    flush.zero_()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    dg.matvec(x, y, form=form)
                    b.record()
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(b))
                t = float(np.mean(ts))
                res[f"{form}_{dtype}"] = {"ms": t, "Gedges_s": g.m / t / 1e6}
                dg.close()
            except Exception as e:  # noqa: BLE001 (report, do not hide)
                res[f"{form}_{dtype}"] = {"error": str(e)[:200]}
    log(json.dumps(res))
    return res


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
