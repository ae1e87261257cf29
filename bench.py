#!/usr/bin/env python
"""Headline benchmark: compressed A·x on B200 (BASELINE.json metric
"compressed A·x Gedges/s ... % HBM roofline ...").

Workload (N=1): BASELINE.json configs[1] (C2): synthetic copy-model graph,
n = 2^24, mean out-degree 20, BV w=7 R=3 Lmin=4 zeta_3, one y = A x^T in fp64
per step with x ~ U[0,1) resident in HBM.  Under torchrun each rank runs its
own C2-sized graph (weak scaling, no data-path collective).

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


def make_workload(args, rank):
    import paper_1708_07271_b200 as P

    n = 1 << args.n_log2
    t0 = time.time()
    g = P.CsrGraph.copy_model(n, args.degree, 0.7, 0.8, seed=SEED + 2 + 1000 * rank)
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


def cpu_reference_throughput(g, x64, steps, warmup, budget_s, threads=None):
    """The reference's own path restated (oracle): matvec_ref_into on
    compress(g, 7), sequential per product, run as `threads`
    concurrent independent products (SPEC.md:228 allows that) on the host
    cores.  Returns (edges/s, sample description, cores, per-step values)."""
    from oracle import pyoracle as O

    threads = threads or O.threads()
    t0 = time.time()
    og = O.Csr.from_arrays(g.n, g.row_offsets, g.columns)
    rm = O.RefMatrix.compress(og, 7, threads)
    tc = time.time() - t0
    log(f"[cpu] compress(g,7) with {threads} threads took {tc:.1f}s")
    vals = []
    t_start = time.time()
    for k in range(warmup + steps):
        sec = rm.matvec_concurrent(x64, threads)
        if k >= warmup:
            vals.append(threads * g.m / sec)
        if time.time() - t_start > budget_s and len(vals) >= 1:
            break
    sample = (f"{len(vals)} timed rounds of {threads} concurrent full matvec_ref products "
              f"(n={g.n}, m={g.m}) on compress(g,7); compress took {tc:.1f}s")
    return float(np.median(vals)), sample, threads, vals


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU reference
    import paper_1708_07271_b200 as P  # generator only (host C++)

    g, _ = make_workload(args, 0)
    x64 = x_uniform(g.n, 11, "f64")
    v, sample, cores, _ = cpu_reference_throughput(g, x64, args.steps, args.warmup, budget_s=1e9)
    gv = v / 1e9
    out = {
        "metric": "compressed A·x Gedges/s", "value": gv, "unit": "Gedges/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": g.m / v * 1e3 * cores,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": f"C2 copy-model n=2^{args.n_log2} deg{args.degree:g} y=A·x^T fp64 "
                               f"(BASELINE.json configs[1])",
                   "n": g.n, "m": g.m, "reference_format": "compress(g,7) A' (ref_matrix.hpp:69)"},
        "cpu_baseline": {"value": gv, "unit": "Gedges/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": gv, "unit": "Gedges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1708_07271_b200 as P

    rank, world, local = dist_env()
    if world != args.gpus:
        args.gpus = world
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    g, s = make_workload(args, rank)
    opts = P.CreateOptions(device=local, block_rows=args.block_rows, lanes=args.lanes, window=args.window)
    t0 = time.time()
    dg = P.BvGraph(s, opts)
    info = dg.info()
    log(f"[rank {rank}] device handle built in {time.time() - t0:.1f}s: {info}")
    S = s.stats()["stream_bits"]
    xsz = 8 if args.dtype == "f64" else 4
    xh = x_uniform(g.n, 11 + rank, args.dtype)
    x = torch.from_numpy(xh).to(dev)
    y = torch.empty(g.n, dtype=x.dtype, device=dev)
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
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for k in range(args.steps):
        flush.zero_()  # L2 flush between timed iterations (outside the events)
        evs[k][0].record(stream)
        step()
        evs[k][1].record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    keep_busy(0.4)
    clocks = sampler.stop()
    if clocks is not None:
        clocks["how"] = "nvidia-smi -lms 50 across warm-up, the timed steps and surrounding identical untimed launches"
    times = np.array([a.elapsed_time(b) for a, b in evs])  # ms per launch
    t_mean = float(times.mean())
    if world > 1:
        tt = torch.tensor([t_mean], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_mean = float(tt.item())
    m_total = g.m  # edges processed per step by all ranks (each rank has its own graph)
    if world > 1:
        mt = torch.tensor([float(g.m)], device=dev, dtype=torch.float64)
        dist.all_reduce(mt, op=dist.ReduceOp.SUM)
        m_total = float(mt.item())
    value = m_total / (t_mean * 1e-3) / 1e9

    # roofline of the dominant (only) kernel: algorithmic bytes per launch
    alg_bytes = math.ceil(S / 8) + g.n * xsz + g.n * xsz
    peak, peak_src = measured_peak()
    achieved = alg_bytes / (float(times.mean()) * 1e-3) / 1e9
    traffic = None  # dram bytes per launch of this kernel from the committed ncu --set full capture
    prof = os.path.join(ROOT, "profiles", "ncu_gather_summary.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            key = f"{args.form}_{args.dtype}_n{args.n_log2}_t{args.lanes}_w{args.window}"
            if key in pj:
                traffic = pj[key]["dram_bytes_per_launch"]
        except Exception:
            traffic = None

    # e2e through the C-ABI host-pointer path (H2D + kernel + D2H each step)
    e2e = None
    if not args.no_e2e:
        xpin = torch.from_numpy(xh).pin_memory().numpy()
        ypin = torch.empty(g.n, dtype=x.dtype).pin_memory().numpy()
        for _ in range(max(1, args.warmup // 2)):
            dg.matvec(xpin, ypin, form=args.form)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        e_times = []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            dg.matvec(xpin, ypin, form=args.form)  # synchronous: copies + kernel
            e_times.append(time.perf_counter() - t0)
        te = float(np.mean(e_times))
        if world > 1:
            tt = torch.tensor([te], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": m_total / te / 1e9, "unit": "Gedges/s", "h2d_bytes_per_step": g.n * xsz,
               "d2h_bytes_per_step": g.n * xsz, "ms_per_step": te * 1e3,
               "how": "cmvg_matvec_* with HOST pointers (pinned); wall clock around the synchronous call"}

    # correctness spot check against the oracle's matvec_csr (rank 0, outside timing)
    parity = None
    if rank == 0:
        from oracle import pyoracle as O
        want = O.matvec_csr_raw(g.n, g.row_offsets, g.columns, np.ascontiguousarray(xh, dtype=np.float64),
                                O.threads())
        got = y.double().cpu().numpy() if args.form == "gather" else None
        if got is not None:
            nz = want != 0
            parity = float(np.max(np.abs(got[nz] - want[nz]) / np.abs(want[nz])))

    # uncompressed comparison point at equal hardware: the reference's
    # matvec_csr as a hand-written CSR kernel on the same GPU (PAPER.md:217's
    # S = t/t'), same x, same L2 flush; rank 0, outside the timed region
    csr_base = None
    if rank == 0 and args.form == "gather" and args.dtype == "f64" and not args.no_csr:
        ro = torch.from_numpy(g.row_offsets.astype(np.int64)).to(dev)
        co = torch.from_numpy(g.columns.view(np.int32)).to(dev)
        yc = torch.empty_like(x)
        for _ in range(args.warmup):
            flush.zero_()
            P.csr_matvec_device(ro, co, x, yc, stream=stream.cuda_stream)
        cevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for a, b in cevs:
            flush.zero_()
            a.record(stream)
            P.csr_matvec_device(ro, co, x, yc, stream=stream.cuda_stream)
            b.record(stream)
        torch.cuda.synchronize(dev)
        tc = float(np.mean([a.elapsed_time(b) for a, b in cevs]))
        csr_bytes = 4 * g.m + 8 * (g.n + 1) + 16 * g.n
        pk, _ = measured_peak()
        csr_base = {"ms": tc, "gedges_s": g.m / (tc * 1e-3) / 1e9, "bv_speedup": tc / float(times.mean()),
                    "bytes_per_launch": csr_bytes, "gbs": csr_bytes / (tc * 1e-3) / 1e9,
                    "roofline_ms": csr_bytes / (pk * 1e9) * 1e3,
                    "bv_speedup_vs_csr_roofline": csr_bytes / (pk * 1e9) / (float(times.mean()) * 1e-3),
                    "what": "hand-written GPU CSR product (u64 row offsets, u32 columns, fp64; matvec_csr, "
                            "csr.hpp:48-55) on the same B200: bv_speedup = t_csr / t_compressed, the paper's "
                            "S = t/t' (PAPER.md:217) at equal hardware; roofline_ms = the CSR bytes at peak HBM "
                            "bandwidth (an ideal CSR kernel), bv_speedup_vs_csr_roofline = roofline_ms / t_compressed"}
        if parity is not None:
            wc = yc.cpu().numpy()
            nz = want != 0
            csr_base["parity_max_rel_err"] = float(np.max(np.abs(wc[nz] - want[nz]) / np.abs(want[nz])))
        del ro, co, yc

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        x64 = np.ascontiguousarray(xh, dtype=np.float64)
        v, sample, cores, _ = cpu_reference_throughput(g, x64, steps=3, warmup=1, budget_s=args.cpu_sample_seconds)
        cpu = {"value": v / 1e9, "unit": "Gedges/s", "cores": cores, "kind": "port", "sample": sample}

    secondary = {}
    if args.secondary and rank == 0:
        secondary = run_secondary(args, g, s, dev)

    if rank == 0:
        out = {
            "metric": "compressed A·x Gedges/s", "value": value, "unit": "Gedges/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_mean, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": {
                "workload": f"C2 copy-model n=2^{args.n_log2} deg{args.degree:g} y=A·x^T ({args.form}) "
                            f"{args.dtype} (BASELINE.json configs[1]); each rank its own graph",
                "n": g.n, "m": g.m, "bv": "w=7 R=3 Lmin=4 zeta3 segment=1024",
                "S_bits": S, "bits_per_edge": S / g.m,
                "device_layout": "BV-S (sliced)" if args.form == "gather" else "BV-D",
                "device_layout_bytes": (info["bvs_stream_bytes"] if args.form == "gather" else info["bvd_stream_bytes"])
                + info["bvd_block_table_bytes"],
                "block_rows": args.block_rows, "lanes": args.lanes, "window": args.window,
                "l2": "flushed (512 MiB write) before every timed launch",
                "parallelism": f"weak replicas x{world}",
            },
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "alg_bytes_per_launch": alg_bytes,
                         "alg_bytes_formula": "ceil(S/8) + n*sizeof(x) + n*sizeof(y)"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": args.steps,
            "clocks": clocks,
            "parity_max_rel_err_vs_matvec_csr": parity,
            "csr_baseline": csr_base,
            "kernel_ms": {"mean": float(times.mean()), "median": float(np.median(times)),
                          "min": float(times.min()), "max": float(times.max())},
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
