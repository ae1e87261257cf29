"""Full-size evidence for BASELINE.json configs 1-5 (GPU box): generate each
config, BV-encode it, run the device product(s), check parity against the CPU
oracle at FULL size, and time the kernels with CUDA events.

    python tools/run_configs.py [--configs 1,2,3,4,5] [--out profiles/configs_r1.json]

Parity bars (north_star): decoded adjacency bit-exact; fp64 <= 1e-12 and
fp32 <= 1e-5 relative per entry vs the oracle's matvec_csr (fp64, on the
fp32-rounded input for fp32); PageRank <= 1e-12 relative per entry vs the
oracle's pagerank(CsrKernel(A^T)) with sum p = 1 within 1e-10.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1708_07271_b200 as P  # noqa: E402
from oracle import pyoracle as O  # noqa: E402

SEED = 0x170807271


def measured_peak():
    """HBM GB/s from MEASURED_PEAKS.json (driver-written), else the profiling recipe's fallback."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


PEAK = measured_peak()


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def rel_err(y, want):
    y = np.asarray(y, dtype=np.float64)
    nz = want != 0
    if np.any(y[~nz] != 0):
        return float("inf")
    return float(np.max(np.abs(y[nz] - want[nz]) / np.abs(want[nz]))) if nz.any() else 0.0


def xu(n, seed, k=None):
    rng = np.random.default_rng(seed)
    shape = (n,) if k is None else (n, k)
    return (rng.integers(0, 2**64, size=shape, dtype=np.uint64) >> np.uint64(11)).astype(np.float64) * 2.0**-53


def time_launch(fn, reps=10, flush=None):
    ts = []
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return float(np.median(ts))


def graph(cfg, n):
    if cfg == 4:
        return P.CsrGraph.social(n, seed=SEED + 4)
    deg = {1: 12.0, 2: 20.0, 3: 24.0, 5: 16.0}[cfg]
    return P.CsrGraph.copy_model(n, deg, 0.7, 0.8, seed=SEED + cfg)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "configs_r2.json"))
    ap.add_argument("--scale", type=int, default=0, help="subtract from every n_log2 (quick runs)")
    args = ap.parse_args()
    res = {"gpu": torch.cuda.get_device_name(0), "host_threads": O.threads()}
    flush = torch.empty(128 << 20, dtype=torch.int32, device="cuda")
    th = O.threads()
    for cfg in [int(c) for c in args.configs.split(",")]:
        nlog = {1: 20, 2: 24, 3: 26, 4: 25, 5: 27}[cfg] - args.scale
        n = 1 << nlog
        r = {"n": n}
        t0 = time.time()
        g = graph(cfg, n)
        r["m"] = g.m
        r["gen_s"] = time.time() - t0
        log(f"C{cfg}: n=2^{nlog} m={g.m} generated in {r['gen_s']:.1f}s")
        if cfg == 3:
            t0 = time.time()
            at = g.transpose()
            r["transpose_s"] = time.time() - t0
            src = at
        else:
            src = g
        params = P.BvParams(max_ref=0 if cfg == 4 else 3)
        t0 = time.time()
        s = P.BvStream.encode(src, params)
        st = s.stats()
        r["encode_s"] = time.time() - t0
        r["S_bits"] = st["stream_bits"]
        r["bits_per_edge"] = st["stream_bits"] / g.m
        r["max_depth"] = st["max_depth"]
        t0 = time.time()
        dg = P.BvGraph(s, P.CreateOptions(window=3968 if cfg == 4 else 1536))  # C4: community-sized window
        r["handle_s"] = time.time() - t0
        info = dg.info()
        r["device_layout"] = "BV-F (gather, PageRank)"
        r["device_layout_bytes"] = info["bvf_stream_bytes"] + info["bvd_block_table_bytes"]
        r["bvf_terms"] = info["bvf_terms"]
        r["bvf_pad_terms"] = info["bvf_pad_terms"]
        r["bvf_esc_terms"] = info["bvf_esc_terms"]
        r["window_coverage"] = info["window_coverage"]
        ro = src.row_offsets
        co = src.columns
        # decoded adjacency, bit-exact (GPU BV decoder)
        drp = torch.empty(src.n + 1, dtype=torch.int64, device="cuda")
        dco = torch.empty(max(src.m, 1), dtype=torch.int32, device="cuda")
        t = time_launch(lambda: dg.decode_csr_device(drp, dco), reps=2)
        ok = bool(np.array_equal(drp.cpu().numpy().view(np.uint64), ro)) and bool(
            np.array_equal(dco[: src.m].cpu().numpy().view(np.uint32), co))
        r["decode_csr"] = {"bit_exact": ok, "s": t}
        del drp, dco
        S8 = st["stream_bits"] / 8
        if cfg in (1, 2, 4):
            x = xu(n, 11)
            for dt, tol in (("f64", 1e-12), ("f32", 1e-5)):
                if cfg == 4 and dt == "f64":
                    continue
                xh = x if dt == "f64" else x.astype(np.float32)
                xd = torch.from_numpy(xh).cuda()
                yd = torch.empty_like(xd)
                want = O.matvec_csr_raw(n, ro, co, xh.astype(np.float64), th)
                tg = time_launch(lambda: dg.matvec(xd, yd), flush=flush)
                e = rel_err(yd.double().cpu().numpy(), want)
                alg = S8 + 2 * n * xh.itemsize
                r[f"gather_{dt}"] = {"s": tg, "Gedges_s": g.m / tg / 1e9, "max_rel_err": e, "tol": tol,
                                     "pass": bool(e <= tol), "roofline_frac": alg / tg / 1e9 / PEAK}
                if cfg == 2:
                    og = O.Csr.from_arrays(n, ro, co).transpose()
                    wl = og.matvec(xh.astype(np.float64), th)
                    del og
                    ts_ = time_launch(lambda: dg.matvec(xd, yd, form="scatter"), flush=flush)
                    r["bvt_stream_bytes"] = dg.info()["bvt_stream_bytes"]
                    e = rel_err(yd.double().cpu().numpy(), wl)
                    r[f"scatter_{dt}"] = {"s": ts_, "Gedges_s": g.m / ts_ / 1e9, "max_rel_err": e, "tol": tol,
                                          "pass": bool(e <= tol), "roofline_frac": alg / ts_ / 1e9 / PEAK}
                    # x A the reference's way: (A^T) x on the transpose's compression, built on the GPU
                    t0 = time.time()
                    dg.matvec(xd, yd, form="left")
                    torch.cuda.synchronize()
                    first = time.time() - t0
                    ts_ = time_launch(lambda: dg.matvec(xd, yd, form="left"), flush=flush)
                    e = rel_err(yd.double().cpu().numpy(), wl)
                    r[f"left_{dt}"] = {"s": ts_, "Gedges_s": g.m / ts_ / 1e9, "max_rel_err": e, "tol": tol,
                                       "pass": bool(e <= tol), "roofline_frac": alg / ts_ / 1e9 / PEAK,
                                       "first_call_s (A^T layout built on the GPU)": first}
                del xd, yd
        if cfg == 3:
            deg = g.out_degrees()
            degd = torch.from_numpy(deg.astype(np.int32)).cuda()
            dg.pagerank(degd, alpha=0.15, iterations=4, dangling="uniform")  # warm-up (allocations, graph capture)
            torch.cuda.synchronize()
            t0 = time.time()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            p, it = dg.pagerank(degd, alpha=0.15, iterations=50, dangling="uniform")
            b.record()
            torch.cuda.synchronize()
            tpr = a.elapsed_time(b) * 1e-3
            og = O.Csr.from_arrays(n, ro, co)
            t0 = time.time()
            want, wit = O.pagerank_csr(og, deg, 0.15, 50, dangling="uniform", nthreads=th)
            r["oracle_pagerank_s"] = time.time() - t0
            pn = p.cpu().numpy()
            e = rel_err(pn, want)
            alg = S8 + n * (8 + 8 + 4) * 50 / 50
            r["pagerank"] = {"iterations": int(it), "s": tpr, "iter_per_s": it / tpr, "max_rel_err": e, "tol": 1e-12,
                             "sum_minus_1": float(abs(pn.sum() - 1.0)), "pass": bool(e <= 1e-12 and abs(pn.sum() - 1) <= 1e-10),
                             "roofline_frac_per_iter": (S8 + n * 28) / (tpr / it) / 1e9 / PEAK,
                             "alg_bytes_per_iter": "ceil(S/8) + 8n (q) + 8n (p) + 8n (q') + 4n (d)"}
            del og
        if cfg == 5:
            k = 16
            X = xu(n, 13, k).astype(np.float32)
            Xd = torch.from_numpy(X).cuda()
            Yd = torch.empty_like(Xd)
            tm = time_launch(lambda: dg.matmat(Xd, Yd), reps=5, flush=flush)
            r["bvs_stream_bytes"] = dg.info()["bvs_stream_bytes"]
            Y = Yd.cpu().numpy()
            errs = []
            for c in range(k):
                want = O.matvec_csr_raw(n, ro, co, np.ascontiguousarray(X[:, c], dtype=np.float64), th)
                errs.append(rel_err(Y[:, c], want))
            e = max(errs)
            alg = S8 + 2 * n * k * 4
            r["matmat_f32_k16"] = {"s": tm, "Gedge_vectors_s": g.m * k / tm / 1e9, "max_rel_err": e, "tol": 1e-5,
                                   "pass": bool(e <= 1e-5), "roofline_frac": alg / tm / 1e9 / PEAK}
            del Xd, Yd
        res[f"C{cfg}"] = r
        log(json.dumps(r))
        del dg, s, g, src
        torch.cuda.empty_cache()
        json.dump(res, open(args.out, "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
